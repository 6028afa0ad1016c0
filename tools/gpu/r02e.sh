python tools/oz_pass.py 200000 20000 256 0 3 > gpurun_out/oz_pass.txt 2>&1
python tools/oz_pass.py 50000 20000 256 0 1 >> gpurun_out/oz_pass.txt 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:"ozaki_gemm" -c 1 -o /tmp/oz_nn python tools/oz_pass.py 50000 20000 256 0 1 > gpurun_out/ncu_oz.log 2>&1
ncu -i /tmp/oz_nn.ncu-rep --page details --csv > gpurun_out/ncu_oz_nn_details.csv 2>/dev/null
ncu -i /tmp/oz_nn.ncu-rep --page raw --csv > gpurun_out/ncu_oz_nn_raw.csv 2>/dev/null
ncu -i /tmp/oz_nn.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_oz_nn_source.csv 2>/dev/null
cp /tmp/oz_nn.ncu-rep gpurun_out/
echo done
