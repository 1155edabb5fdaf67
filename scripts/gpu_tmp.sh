mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r01o_bench.json 2> gpurun_out/r01o_bench.err; echo "bench $?"
python -c "
import json; d=json.load(open('gpurun_out/r01o_bench.json')); print('products', d['ms_per_step'], d['value']/1e9, {k:(round(v['ms'],1),v['calls']) for k,v in d['kernels'].items()})"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "layer_parity or variants" > gpurun_out/r01o_tests.log 2>&1; echo "tests $?"; tail -2 gpurun_out/r01o_tests.log
