timeout 600 python tools/oz_check.py > gpurun_out/oz_check.txt 2>&1
echo "rc=$?"
python tools/oz_pass.py 200000 20000 256 0 3 > gpurun_out/oz_pass.txt 2>&1
python tools/oz_pass.py 200000 20000 256 1 3 >> gpurun_out/oz_pass.txt 2>&1
