set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 -p no:cacheprovider > gpurun_out/pytest_r02q.log 2>&1
echo "pytest rc=$?"
tail -25 gpurun_out/pytest_r02q.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02q.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_r02q.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c3_r02q.json 2> gpurun_out/bench_c3_r02q.err
echo "bench rc=$?"
head -c 4000 gpurun_out/bench_c3_r02q.json
