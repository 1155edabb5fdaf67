# one ncu --set full capture of the products phase; per-kernel source pages of the NN GEMM and
# the main SpMM (stall sampling), summaries into gpurun_out/
mkdir -p gpurun_out
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -o /tmp/phase_full python scripts/ncu_phase.py products bf16 gpurun_out/ncu_phase_calls.json > gpurun_out/ncu_phase.log 2>&1
tail -2 gpurun_out/ncu_phase.log
python scripts/ncu_summary.py full /tmp/phase_full.ncu-rep --calls gpurun_out/ncu_phase_calls.json > gpurun_out/ncu_summary_phase.json
ncu -i /tmp/phase_full.ncu-rep --page details --csv > gpurun_out/phase_details.csv 2>/dev/null
ncu -i /tmp/phase_full.ncu-rep --page source --csv -k regex:k_gemm_tc_nn -c 1 > gpurun_out/gemm_source.csv 2>/dev/null
ncu -i /tmp/phase_full.ncu-rep --page source --csv -k regex:k_spmm_grp -c 1 > gpurun_out/spmm_source.csv 2>/dev/null
ncu -i /tmp/phase_full.ncu-rep --page raw --csv -k regex:k_gemm_tc_nn -c 1 > gpurun_out/gemm_raw.csv 2>/dev/null
ls -la gpurun_out | tail -8
