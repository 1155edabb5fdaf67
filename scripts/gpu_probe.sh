# one gpurun call: roofline probes + ncu LTS/DRAM metrics of the gather probe and of the SpMM
mkdir -p gpurun_out
timeout 300 python scripts/roofline_probe.py gpurun_out/probe.json > gpurun_out/probe.log 2>&1; echo "probe exit $?"
tail -40 gpurun_out/probe.log
