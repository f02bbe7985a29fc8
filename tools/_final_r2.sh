#!/bin/bash
# End-of-round-2 evidence: parity gate, C5 A/B of the one-CTA routing, the evidence run (smoke, GPU
# suite, all configs, reference arm), the ViT-L/32 step launch list and ncu --set full of its fc1+GELU GEMM.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_kernels_gpu.py tests/test_vit_gpu.py -q -p no:cacheprovider -x > gpurun_out/f_tests.log 2>&1
tail -3 gpurun_out/f_tests.log
grep -q " passed" gpurun_out/f_tests.log && ! grep -q "failed\|error" gpurun_out/f_tests.log || exit 1
summ() { tail -1 $1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('value', d['value'], 'nofreeze', d['nofreeze']['value'], 'ms', d['ms_per_step'], 'roof', d['roofline']['achieved'], 'clk', d['clocks']['sm_mhz'])"; }
PF_GEMM_SMALL_ONECTA=0 PF_SKIP_CPU_BASELINE=1 timeout 600 python bench.py --model vit-l-32 --schedule gpipe --microbatches 8 > gpurun_out/f_c5_pair.log 2>&1; echo "c5 pair"; summ gpurun_out/f_c5_pair.log
PF_SKIP_CPU_BASELINE=1 timeout 600 python bench.py --model vit-l-32 --schedule gpipe --microbatches 8 > gpurun_out/f_c5_onecta.log 2>&1; echo "c5 onecta"; summ gpurun_out/f_c5_onecta.log
bash tools/_evidence.sh
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_vit_launches.csv python tools/profile_step.py --model vit-l-32 --ratio 0.8 > gpurun_out/r2f_vit_prof.log 2>&1
tail -2 gpurun_out/r2f_vit_prof.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tcgen05_pair -s 40 -c 12 -o gpurun_out/r2f_vit_gemm_full -f python tools/profile_step.py --model vit-l-32 --ratio 0.8 > gpurun_out/r2f_vit_full.log 2>&1
tail -2 gpurun_out/r2f_vit_full.log
ls -la gpurun_out | tail -5
