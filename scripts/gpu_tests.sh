# gpurun: the GPU test suite (+ smoke); logs under gpurun_out/
mkdir -p gpurun_out
TAG=${1:-r02}
timeout ${TEST_TIMEOUT:-1700} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest gpu exit $?"; tail -15 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke exit $?"; tail -2 gpurun_out/${TAG}_smoke.log
