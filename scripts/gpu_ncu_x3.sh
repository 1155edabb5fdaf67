# ncu --set full of the split-fp32 GEMMs in one products phase (fp32 storage); raw + source pages
mkdir -p gpurun_out
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_gemm_x3 \
  -o /tmp/x3_full python scripts/ncu_phase.py products f32 gpurun_out/ncu_phase_calls_f32.json > gpurun_out/ncu_x3.log 2>&1
tail -2 gpurun_out/ncu_x3.log
python scripts/ncu_summary.py full /tmp/x3_full.ncu-rep --calls gpurun_out/ncu_phase_calls_f32.json > gpurun_out/ncu_summary_x3.json
ncu -i /tmp/x3_full.ncu-rep --page details --csv > gpurun_out/x3_details.csv 2>/dev/null
ncu -i /tmp/x3_full.ncu-rep --page source --csv -k regex:k_gemm_x3_nn -c 1 > gpurun_out/x3nn_source.csv 2>/dev/null
ncu -i /tmp/x3_full.ncu-rep --page raw --csv -k regex:k_gemm_x3_nn -c 1 > gpurun_out/x3nn_raw.csv 2>/dev/null
ls -la gpurun_out | tail -6
