python tools/oz_modes.py c1 c2 c3 c3f32 c5 > gpurun_out/oz_modes.txt 2>&1
