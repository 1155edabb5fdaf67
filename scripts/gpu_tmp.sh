mkdir -p gpurun_out
bash scripts/gpu_round.sh r01x > gpurun_out/r01x_round.log 2>&1; echo "round $?"; tail -45 gpurun_out/r01x_round.log
