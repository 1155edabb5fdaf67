mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python scripts/mb_pipe_check.py 100000 > gpurun_out/r01h_sanitizer.log 2>&1; echo "sanitizer $?"; grep -E "ERROR SUMMARY|OK" gpurun_out/r01h_sanitizer.log | head -5
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01h_gpu.log 2>&1; echo "gpu suite $?"; tail -3 gpurun_out/r01h_gpu.log
timeout 1500 python bench.py --config papers --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01h_bench_papers.json 2> gpurun_out/r01h_bench_papers.err; echo "bench papers $?"; tail -c 300 gpurun_out/r01h_bench_papers.json; tail -3 gpurun_out/r01h_bench_papers.err
timeout 900 python bench.py --dtype f32 > gpurun_out/r01h_bench_products_f32.json 2> gpurun_out/r01h_bench_products_f32.err; echo "bench f32 $?"; tail -c 300 gpurun_out/r01h_bench_products_f32.json
timeout 900 python bench.py --config rmat24 > gpurun_out/r01h_bench_rmat24.json 2> gpurun_out/r01h_bench_rmat24.err; echo "bench rmat24 $?"; tail -c 300 gpurun_out/r01h_bench_rmat24.json; tail -3 gpurun_out/r01h_bench_rmat24.err
timeout 1200 python bench.py --config rmat26 --no-cpu-baseline > gpurun_out/r01h_bench_rmat26.json 2> gpurun_out/r01h_bench_rmat26.err; echo "bench rmat26 $?"; tail -c 300 gpurun_out/r01h_bench_rmat26.json; tail -3 gpurun_out/r01h_bench_rmat26.err
