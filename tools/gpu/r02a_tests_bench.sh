set -x
free -g; nproc; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
export SORSVD_PARITY_OUT=gpurun_out/parity_r02a
timeout 3000 python -m pytest tests -m gpu -q -rf --durations=25 -p no:cacheprovider > gpurun_out/pytest_r02a.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/pytest_r02a.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3_r02a.json 2> gpurun_out/bench_c3_r02a.err
echo "bench rc=$?"
cat gpurun_out/bench_c3_r02a.json | head -c 3000
