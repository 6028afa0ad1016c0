export SORSVD_PARITY_OUT=gpurun_out/parity_r02j
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 -p no:cacheprovider > gpurun_out/pytest_r02j.log 2>&1
echo "pytest rc=$?"
tail -25 gpurun_out/pytest_r02j.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3_r02j.json 2> gpurun_out/bench_c3_r02j.err
echo "bench rc=$?"
head -c 4000 gpurun_out/bench_c3_r02j.json
