export SORSVD_PARITY_OUT=gpurun_out/parity_r02l
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 -p no:cacheprovider > gpurun_out/pytest_r02l.log 2>&1
echo "pytest rc=$?"
tail -14 gpurun_out/pytest_r02l.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3_r02l.json 2> gpurun_out/bench_c3_r02l.err
echo "bench rc=$?"
python tools/profile_stages.py --config c3 --reps 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_r02l.csv python tools/profile_stages.py --config c3 --reps 1 > /dev/null 2>&1
echo "ncu launches rc=$?"
