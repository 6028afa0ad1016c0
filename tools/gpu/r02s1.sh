set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 -p no:cacheprovider > gpurun_out/pytest_r02s1.log 2>&1
echo "pytest rc=$?"
tail -25 gpurun_out/pytest_r02s1.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02s1.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_r02s1.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c3_r02s1.json 2> gpurun_out/bench_c3_r02s1.err
echo "bench rc=$?"
head -c 4000 gpurun_out/bench_c3_r02s1.json
for c in c2 c4 c1; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_${c}_r02s1.json 2> gpurun_out/bench_${c}_r02s1.err; echo "rc=$?"; head -c 2500 gpurun_out/bench_${c}_r02s1.json; done
