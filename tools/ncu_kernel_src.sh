#!/bin/bash
# ncu source-level capture of one kernel (regex $1) of a python command ($2...) -> gpurun_out/<tag>_*.csv
set -u
re=$1; tag=$2; shift 2
mkdir -p gpurun_out
"$@" > /dev/null 2>&1 || { echo "command failed"; exit 1; }
ncu -f --set full --clock-control none --import-source on -k regex:"$re" -c 1 -o /tmp/$tag "$@" > gpurun_out/ncu_$tag.log 2>&1
ncu -i /tmp/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv 2>/dev/null
ncu -i /tmp/$tag.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv 2>/dev/null
ncu -i /tmp/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
echo "captured $tag"
