python tools/dbg_bufs.py > gpurun_out/dbg_bufs.txt 2>&1
