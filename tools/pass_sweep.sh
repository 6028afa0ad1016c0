#!/bin/bash
# Pass-kernel timings (CUDA events, 20 reps) for the main configs -> stdout.
for spec in "c2 0" "c2 1" "c1 0" "c3 0" "c3 1" "c3f32 0" "c3f32 1"; do
  set -- $spec
  timeout 300 python tools/run_pass.py --config $1 --ta $2 --reps 20 2>&1 | tail -1
done
