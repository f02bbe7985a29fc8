cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_kernels_gpu.py tests/test_vit_gpu.py tests/test_northstar_gpu.py -q -p no:cacheprovider -x > gpurun_out/ab3_tests.log 2>&1; tail -3 gpurun_out/ab3_tests.log
summ() { tail -1 $1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('value', d['value'], 'nofreeze', d['nofreeze']['value'], 'ms', d['ms_per_step'], 'roof', d['roofline']['achieved'], 'clk', d['clocks']['sm_mhz'])"; }
echo "== main"; timeout 300 python tools/gelu_bench.py 2>&1 | tail -2; timeout 300 python tools/vit_gemm_bench.py 2>&1 | head -8
PF_SKIP_CPU_BASELINE=1 timeout 600 python bench.py --model vit-l-32 --schedule gpipe --microbatches 8 > gpurun_out/ab3_c5.log 2>&1; summ gpurun_out/ab3_c5.log
PF_SKIP_CPU_BASELINE=1 timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/ab3_c3.log 2>&1; summ gpurun_out/ab3_c3.log
cp paper_2602_05754_b200/lib/libpf_device.so /tmp/main.so
cp ab_variants/libpf_device_store2.so paper_2602_05754_b200/lib/libpf_device.so
echo "== store2"; timeout 300 python tools/vit_gemm_bench.py 2>&1 | head -8
PF_SKIP_CPU_BASELINE=1 timeout 600 python bench.py --model vit-l-32 --schedule gpipe --microbatches 8 > gpurun_out/ab3_c5_s2.log 2>&1; summ gpurun_out/ab3_c5_s2.log
PF_SKIP_CPU_BASELINE=1 timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/ab3_c3_s2.log 2>&1; summ gpurun_out/ab3_c3_s2.log
cp /tmp/main.so paper_2602_05754_b200/lib/libpf_device.so
echo "== main again"; PF_SKIP_CPU_BASELINE=1 timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/ab3_c3b.log 2>&1; summ gpurun_out/ab3_c3b.log
