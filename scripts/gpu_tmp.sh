mkdir -p gpurun_out
for v in "tnstages=4 --variant tnred=8" "tnstages=0 --variant tnred=8" "tnstages=4 --variant tnred=32" "tnstages=0 --variant tnred=32" "tnstages=6 --variant tnred=8"; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --variant $v > gpurun_out/r01v_b.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/r01v_b.json')); print('$v', round(d['ms_per_step'],2), {k:(round(v['ms'],1),v['calls']) for k,v in d['kernels'].items() if k in ('gemm_tn','spmm','gemm')})"
done
