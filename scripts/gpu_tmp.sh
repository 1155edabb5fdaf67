mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_capacity.py -x -q > gpurun_out/r01k_cap.log 2>&1; echo "cap $?"; tail -20 gpurun_out/r01k_cap.log
