# gpurun: a quick subset -- selected GPU tests (PYTEST_K) + optional probes.  Logs in gpurun_out/.
mkdir -p gpurun_out
TAG=${1:-q}
timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest exit $?"; tail -${TAIL:-15} gpurun_out/${TAG}_pytest.log
if [ -n "$REPART" ]; then timeout 300 python scripts/repart_probe.py 3 $REPART > gpurun_out/${TAG}_repart.log 2>&1; echo "repart $?"; tail -4 gpurun_out/${TAG}_repart.log; fi
if [ -n "$BENCH" ]; then GRAPPA_GRAPH_TIMING=1 timeout 900 python bench.py $BENCH > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench $?"; tail -5 gpurun_out/${TAG}_bench.err; python -c "import json,sys; d=json.load(open(sys.argv[1])); print(d['ms_per_step'], d['config']['epoch_ms'], d['config'].get('repartition_ms_per_switch'), (d.get('e2e') or {}).get('ms_per_step'))" gpurun_out/${TAG}_bench.json; fi
