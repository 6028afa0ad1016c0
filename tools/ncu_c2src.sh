set -u
mkdir -p gpurun_out
python tools/run_pass.py --config c2 --ta 0 --reps 20 > gpurun_out/pass_c2.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:gemm_f64_kernel -c 1 -o /tmp/c2nn python tools/run_pass.py --config c2 --ta 0 --reps 1 > gpurun_out/ncu_c2nn.log 2>&1
ncu -i /tmp/c2nn.ncu-rep --page raw --csv > gpurun_out/c2nn_raw.csv 2>/dev/null
ncu -i /tmp/c2nn.ncu-rep --page source --csv --print-source sass > gpurun_out/c2nn_sass.csv 2>/dev/null
ncu -i /tmp/c2nn.ncu-rep --page details --csv > gpurun_out/c2nn_details.csv 2>/dev/null
cp /tmp/c2nn.ncu-rep gpurun_out/
