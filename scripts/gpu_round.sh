# Round check on one B200: GPU parity tests, smoke(), the default bench line (with e2e and the
# oracle cpu_baseline), the reference arm, the ncu launch list of the bench command, and one
# ncu --set full capture of a products phase.  Everything lands in gpurun_out/.
# Usage (from the repo root, via gpurun): bash scripts/gpu_round.sh [tag]
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest gpu exit $?"; tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke exit $?"; tail -2 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench exit $?"; tail -c 600 gpurun_out/${TAG}_bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
echo "ref exit $?"; tail -c 300 gpurun_out/${TAG}_bench_ref.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/${TAG}_bench_under_ncu.log 2>&1
echo "ncu launches exit $?"
python scripts/ncu_summary.py launches gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches.txt 2>&1
head -30 gpurun_out/${TAG}_launches.txt
if [ "${NCU_FULL:-1}" = "1" ]; then
  timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -o /tmp/phase_full python scripts/ncu_phase.py products bf16 gpurun_out/ncu_phase_calls.json \
    > gpurun_out/${TAG}_ncu_phase.log 2>&1
  echo "ncu full exit $?"
  python scripts/ncu_summary.py full /tmp/phase_full.ncu-rep --calls gpurun_out/ncu_phase_calls.json \
    > gpurun_out/${TAG}_ncu_summary.json
  ncu -i /tmp/phase_full.ncu-rep --page details --csv > gpurun_out/${TAG}_phase_details.csv 2>/dev/null
fi
ls -la gpurun_out | tail -20
# side lines (profiles/r01_bench_*.json): every BASELINE config and option the bench offers
if [ "${SIDE:-1}" != "0" ]; then
  nb=--no-cpu-baseline
  SPECS_ALL=1
  for spec in "f32:--dtype f32 $nb" "sharded:--sharded $nb" "halo:--halo $nb" "sharded_halo:--sharded --halo $nb" \
              "node:--corr node $nb" "capshards:--capacity shards $nb" "rmat26_capshards:--config rmat26 --capacity shards $nb" \
              "rmat24:--config rmat24 $nb" "rmat26:--config rmat26 $nb" "arxiv:--config arxiv" "cora:--config cora" \
              "gat:--config products_gat $nb" "capacity:--capacity $nb" "papers:--config papers --steps 4 --warmup 1 $nb"; do
    name=${spec%%:*}; a=${spec#*:}
    timeout 1200 python bench.py $a > gpurun_out/${TAG}_bench_${name}.json 2> gpurun_out/${TAG}_bench_${name}.err
    echo "bench $name exit $?"; python -c "import json,sys; d=json.load(open(sys.argv[1])); c=d['config']; print(d['ms_per_step'], c['epoch_ms']['median'], (d.get('e2e') or {}).get('ms_per_step'), c.get('repartition_ms_per_switch'), c.get('device_mem_peak_gb'))" gpurun_out/${TAG}_bench_${name}.json
  done
fi
