#!/bin/bash
# A/B: TMEM prefetch of the next chunk in the GELU / GELU' epilogues (main) vs HEAD (noprefetch variant).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_kernels_gpu.py tests/test_vit_gpu.py -q -p no:cacheprovider -x > gpurun_out/h_tests.log 2>&1
tail -1 gpurun_out/h_tests.log
grep -q "failed\|error" gpurun_out/h_tests.log && exit 1
summ() { tail -1 $1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('value', d['value'], 'nofreeze', d['nofreeze']['value'], 'ms', d['ms_per_step'], 'roof', d['roofline']['achieved'], 'clk', d['clocks']['sm_mhz'])"; }
for v in main noprefetch main noprefetch; do
  if [ $v = main ]; then cp /tmp/main.so paper_2602_05754_b200/lib/libpf_device.so 2>/dev/null || cp paper_2602_05754_b200/lib/libpf_device.so /tmp/main.so; else cp ab_variants/libpf_device_noprefetch.so paper_2602_05754_b200/lib/libpf_device.so; fi
  echo "== $v"; timeout 300 python tools/gelu_bench.py 2>&1 | tail -2
  PF_SKIP_CPU_BASELINE=1 timeout 600 python bench.py --model vit-l-32 --schedule gpipe --microbatches 8 > gpurun_out/h_c5_$v.log 2>&1; summ gpurun_out/h_c5_$v.log
done
cp /tmp/main.so paper_2602_05754_b200/lib/libpf_device.so
