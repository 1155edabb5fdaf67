# gpurun: diagnostics -- GAT halo debug, the full GPU suite without -x, a switch-timing bench, the
# repartition probe.  Logs under gpurun_out/.
mkdir -p gpurun_out
TAG=${1:-diag}
timeout 300 python scripts/debug/gat_halo_dbg.py > gpurun_out/${TAG}_gat.log 2>&1; echo "gat dbg $?"; tail -20 gpurun_out/${TAG}_gat.log
GRAPPA_GRAPH_TIMING=1 timeout 600 python bench.py --no-cpu-baseline --no-f32 --no-e2e > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench $?"; tail -20 gpurun_out/${TAG}_bench.err; python -c "import json,sys; d=json.load(open(sys.argv[1])); print(d['ms_per_step'], d['config']['epoch_ms'], d['config']['repartition_ms_total'])" gpurun_out/${TAG}_bench.json
timeout 300 python scripts/repart_probe.py 3 products > gpurun_out/${TAG}_repart.log 2>&1; echo "repart $?"; tail -5 gpurun_out/${TAG}_repart.log
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest gpu exit $?"; tail -25 gpurun_out/${TAG}_pytest_gpu.log
