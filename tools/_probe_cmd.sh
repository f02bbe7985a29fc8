cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_flash_attn_gpu.py -q -x 2>&1 | tail -3
echo "== 8b probe"; timeout 150 python tools/step_probe.py --steps 3 2>&1 | tail -4
timeout 1200 python bench.py > gpurun_out/r2e_bench.log 2> gpurun_out/r2e_bench.err; tail -3 gpurun_out/r2e_bench.err; cut -c1-300 gpurun_out/r2e_bench.log
