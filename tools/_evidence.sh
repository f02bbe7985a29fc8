cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z_smoke.log 2>&1; tail -1 gpurun_out/r2z_smoke.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2z_gpu_tests.log 2>&1; tail -1 gpurun_out/r2z_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r2z_bench_c3.log 2> gpurun_out/r2z_bench_c3.err; tail -c 300 gpurun_out/r2z_bench_c3.log
timeout 600 python bench.py --impl reference > gpurun_out/r2z_bench_ref.log 2>&1; tail -c 200 gpurun_out/r2z_bench_ref.log
PF_SKIP_CPU_BASELINE=1 timeout 600 python bench.py --model llama-1b --schedule gpipe --microbatches 8 > gpurun_out/r2z_bench_c2.log 2> gpurun_out/r2z_bench_c2.err; tail -c 200 gpurun_out/r2z_bench_c2.log
PF_SKIP_CPU_BASELINE=1 timeout 600 python bench.py --model vit-l-32 --schedule gpipe --microbatches 8 > gpurun_out/r2z_bench_c5.log 2> gpurun_out/r2z_bench_c5.err; tail -c 200 gpurun_out/r2z_bench_c5.log
PF_SKIP_CPU_BASELINE=1 timeout 900 python bench.py --model llama-13b --layers 5 --schedule interleaved-1f1b --chunks 2 --microbatches 32 > gpurun_out/r2z_bench_c4.log 2> gpurun_out/r2z_bench_c4.err; tail -c 200 gpurun_out/r2z_bench_c4.log
