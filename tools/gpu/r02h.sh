python tools/oz_race.py > gpurun_out/oz_race.txt 2>&1
