timeout 600 python tools/oz_check.py > gpurun_out/oz_check.txt 2>&1
for d in 0 1 6 7; do python tools/oz_pass.py 100000 20000 256 0 3 $d; done > gpurun_out/oz_dbg.txt 2>&1
for d in 0 7; do python tools/oz_pass.py 100000 20000 256 1 3 $d; done >> gpurun_out/oz_dbg.txt 2>&1
