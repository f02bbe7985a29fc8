cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2y_smoke.log 2>&1; tail -1 gpurun_out/r2y_smoke.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2y_gpu_tests.log 2>&1; tail -1 gpurun_out/r2y_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r2y_bench_c3.log 2> gpurun_out/r2y_bench_c3.err; tail -c 300 gpurun_out/r2y_bench_c3.log
PF_SKIP_CPU_BASELINE=1 timeout 600 python bench.py --model vit-l-32 --schedule gpipe --microbatches 8 > gpurun_out/r2y_bench_c5.log 2> gpurun_out/r2y_bench_c5.err; tail -c 200 gpurun_out/r2y_bench_c5.log
timeout 300 python tools/vit_gemm_bench.py > gpurun_out/r2y_vit_gemm.txt 2>&1; tail -30 gpurun_out/r2y_vit_gemm.txt
