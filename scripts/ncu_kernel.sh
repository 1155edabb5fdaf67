# ncu --set full of one launch of a kernel (regex $1) in `python $2...`; summaries into gpurun_out/$3_*
K=$1; shift; TAG=$1; shift
timeout 900 ncu -f --clock-control none -k regex:$K --launch-skip ${SKIP:-2} --launch-count 1 --set full --import-source on -o /tmp/$TAG "$@" > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i /tmp/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>&1
ncu -i /tmp/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>&1
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_source.csv 2>&1
ls -la gpurun_out/${TAG}_*
