set -x
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python tools/profile_step.py --model llama-1b --ratio 0.8 > gpurun_out/prof_launch.log 2>&1
tail -3 gpurun_out/prof_launch.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tcgen05 -s 2 -c 3 -o gpurun_out/gemm_full_r1 python tools/profile_step.py --model llama-1b --ratio 0.8 > gpurun_out/prof_full.log 2>&1
tail -3 gpurun_out/prof_full.log
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:masked_sgd -c 1 -o gpurun_out/optim_full_r1 python tools/profile_step.py --model llama-1b --ratio 0.8 > gpurun_out/prof_opt.log 2>&1
tail -3 gpurun_out/prof_opt.log
ls -la gpurun_out
