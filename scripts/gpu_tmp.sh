mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edge_cases.py -x -q > gpurun_out/r01s_edge.log 2>&1; echo "edge $?"; tail -30 gpurun_out/r01s_edge.log
