#!/bin/bash
# ncu evidence for the C3 bench line with the Ozaki planes engine: launch list of two C3 calls
# (tools/run_config.py c3) and one --set full capture of the NN / TN pass kernels and the
# conversion kernel at full size (tools/oz_pass.py).
set -u
mkdir -p gpurun_out
python tools/run_config.py c3 > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c3_planes.csv \
    python tools/run_config.py c3 > /dev/null 2>&1
for ta in 0 1; do
  ncu -f --set full --clock-control none --import-source on -k regex:"ozaki_planes_gemm|ozaki_rowplanes" -c 2 \
      -o /tmp/c3_planes_ta$ta python tools/oz_pass.py 200000 20000 256 $ta 1 > gpurun_out/ncu_c3_planes_ta$ta.log 2>&1
  echo "ncu ta=$ta rc=$?"
  ncu -i /tmp/c3_planes_ta$ta.ncu-rep --page raw --csv > gpurun_out/r02_ncu_c3_planes_ta${ta}_raw.csv 2>/dev/null
  ncu -i /tmp/c3_planes_ta$ta.ncu-rep --page details --csv > gpurun_out/r02_ncu_c3_planes_ta${ta}_details.csv 2>/dev/null
done
