cd $GRAFT_REPO_ROOT
echo "== default"; timeout 300 python tools/attn_bench.py --iters 20 2>&1 | tail -3
echo "== prof"; PF_ATTN_PROF=1 timeout 300 python tools/attn_bench.py --iters 5 2>&1 | grep -v "^llama.*ours"
echo "== no dQ reductions"; PF_ATTN_PROF=3 timeout 300 python tools/attn_bench.py --iters 20 2>&1 | grep -v cycles
echo "== err"; timeout 300 python tools/attn_err.py 2>&1 | tail -5
