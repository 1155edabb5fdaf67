mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gat.py -x -q > gpurun_out/r01l_gat.log 2>&1; echo "gat $?"; tail -40 gpurun_out/r01l_gat.log
