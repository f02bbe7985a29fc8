#!/bin/bash
# C5 (ViT-L/32) evidence after the one-wave routing fix: parity gate, bench, step launch list, fc1+GELU ncu.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_kernels_gpu.py tests/test_vit_gpu.py -q -p no:cacheprovider -x > gpurun_out/g_tests.log 2>&1
tail -1 gpurun_out/g_tests.log
grep -q "failed\|error" gpurun_out/g_tests.log && exit 1
PF_SKIP_CPU_BASELINE=1 timeout 600 python bench.py --model vit-l-32 --schedule gpipe --microbatches 8 > gpurun_out/r2z_bench_c5.log 2> gpurun_out/r2z_bench_c5.err; tail -c 300 gpurun_out/r2z_bench_c5.log
PF_GEMM_SMALL_ONECTA=0 PF_SKIP_CPU_BASELINE=1 timeout 600 python bench.py --model vit-l-32 --schedule gpipe --microbatches 8 > gpurun_out/g_c5_pair.log 2>&1; tail -c 300 gpurun_out/g_c5_pair.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_vit_launches.csv python tools/profile_step.py --model vit-l-32 --ratio 0.8 > gpurun_out/r2f_vit_prof.log 2>&1
tail -1 gpurun_out/r2f_vit_prof.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tcgen05_pair -s 40 -c 12 -o gpurun_out/r2f_vit_gemm_full -f python tools/profile_step.py --model vit-l-32 --ratio 0.8 > gpurun_out/r2f_vit_full.log 2>&1
tail -1 gpurun_out/r2f_vit_full.log
