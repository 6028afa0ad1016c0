#!/bin/bash
# All bench configurations (one JSON line each) into gpurun_out/; run on the GPU box.
set -u
mkdir -p gpurun_out
for c in c2 c1 c3 c3f32 c3tf32; do
  timeout 1200 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"
done
timeout 1500 python bench.py --config c5 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo "c5 rc=$?"
timeout 900 python bench.py --config c5tf32 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c5tf32.json 2> gpurun_out/bench_c5tf32.err
echo "c5tf32 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
echo "ref rc=$?"
