#!/bin/bash
# C3 end-of-round evidence with the full-M raster: GEMM / north-star parity, the bench line (with
# cpu_baseline), and ncu --set full of the roofline kernel (gate|up + SwiGLU) in the timed step.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_northstar_gpu.py tests/test_stage_gpu.py -q -p no:cacheprovider -x > gpurun_out/j_tests.log 2>&1
tail -1 gpurun_out/j_tests.log
grep -q "failed\|error" gpurun_out/j_tests.log && exit 1
timeout 900 python bench.py > gpurun_out/r2z_bench_c3.log 2> gpurun_out/r2z_bench_c3.err; tail -c 300 gpurun_out/r2z_bench_c3.log
export PF_NCU_RANGE=1 PF_SKIP_CPU_BASELINE=1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  --kernel-name-base mangled -k regex:Li256ELb0ELi4EE -c 1 -o gpurun_out/r2z_roofline -f python bench.py --steps 1 --warmup 3 > gpurun_out/r2z_prof_roof.log 2>&1
tail -1 gpurun_out/r2z_prof_roof.log | cut -c1-200
