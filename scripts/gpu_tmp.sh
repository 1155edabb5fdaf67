mkdir -p gpurun_out
free -g | head -2
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/r01r_full.log 2>&1; echo "full $?"; tail -30 gpurun_out/r01r_full.log
