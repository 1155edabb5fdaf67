mkdir -p gpurun_out
timeout 900 python bench.py --config cora --graph > gpurun_out/r01q_bench_cora.json 2> gpurun_out/r01q_bench_cora.err; echo "cora $?"; tail -3 gpurun_out/r01q_bench_cora.err
python -c "
import json; d=json.load(open('gpurun_out/r01q_bench_cora.json')); print('cora', d['ms_per_step'], d['value']/1e9, (d.get('cpu_baseline') or {}).get('value'))"
timeout 900 python bench.py --config cora4 --graph > gpurun_out/r01q_bench_cora4.json 2> gpurun_out/r01q_bench_cora4.err; echo "cora4 $?"; tail -3 gpurun_out/r01q_bench_cora4.err
python -c "
import json; d=json.load(open('gpurun_out/r01q_bench_cora4.json')); print('cora4', d['ms_per_step'], d['value']/1e9, (d.get('cpu_baseline') or {}).get('value'))"
