#!/bin/bash
# ncu evidence for profiles/: launch list of one C2 call, full captures of the pass kernels
# (summarised to CSV on the box; only the C2 NN report itself is kept).
set -u
mkdir -p gpurun_out
python tools/run_config.py c2 > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/run_config.py c2 > /dev/null 2>&1
for spec in "c2 0" "c2 1" "c3 0" "c3tf32 0"; do
  set -- $spec
  python tools/run_pass.py --config $1 --ta $2 --reps 2 > /dev/null 2>&1 || { echo "pass $1 failed"; continue; }
  rep=/tmp/pass_$1_ta$2
  ncu -f --set full --clock-control none --import-source on -k regex:"gemm_f64_kernel|tc_gemm_tf32" -c 1 \
      -o $rep python tools/run_pass.py --config $1 --ta $2 --reps 1 > gpurun_out/ncu_pass_$1_ta$2.log 2>&1
  echo "ncu $1 ta=$2 rc=$?"
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/ncu_pass_$1_ta$2_raw.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page details --csv > gpurun_out/ncu_pass_$1_ta$2_details.csv 2>/dev/null
done
cp /tmp/pass_c2_ta0.ncu-rep gpurun_out/ 2>/dev/null
du -sh gpurun_out
