mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k normalised > gpurun_out/r01c_fix.log 2>&1; echo "fix $?"; tail -2 gpurun_out/r01c_fix.log
timeout 1500 python scripts/mb_trace.py papers 40 > gpurun_out/r01c_mb_papers.log 2>&1; echo "mb $?"; tail -25 gpurun_out/r01c_mb_papers.log
