python bench.py --config c4 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c4_r02m.json 2>gpurun_out/bench_c4_r02m.err
python bench.py --config c2 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c2_r02m.json 2>gpurun_out/bench_c2_r02m.err
python bench.py --config c1 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c1_r02m.json 2>gpurun_out/bench_c1_r02m.err
python tools/one_c4.py > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_r02m.csv python tools/one_c4.py > /dev/null 2>&1
echo done
