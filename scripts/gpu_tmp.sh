mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01w_gpu.log 2>&1; echo "gpu suite $?"; tail -4 gpurun_out/r01w_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r01w_bench.json 2> gpurun_out/r01w_bench.err; echo "bench $?"; tail -2 gpurun_out/r01w_bench.err
python -c "
import json; d=json.load(open('gpurun_out/r01w_bench.json')); print('products', d['ms_per_step'], d['value']/1e9, d['e2e']['ms_per_step'], {k:(round(v['ms'],1),v['calls']) for k,v in d['kernels'].items()})"
