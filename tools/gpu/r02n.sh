timeout 1500 python -m pytest tests -m gpu -q -rf -x -p no:cacheprovider --deselect tests/test_gpu_fullsize.py > gpurun_out/pytest_r02n.log 2>&1
echo "rc=$?"; tail -5 gpurun_out/pytest_r02n.log
python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4_r02n.json 2>/dev/null
python bench.py --config c1 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_c1_r02n.json 2>/dev/null
python bench.py --config c2 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_c2_r02n.json 2>/dev/null
python tools/one_c4.py > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_r02n.csv python tools/one_c4.py > /dev/null 2>&1
