set -x
python tools/dbg_jacobi_nan.py 150 200 256 > gpurun_out/dbg_jacobi_nan2.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_multirank.py -q -x -p no:cacheprovider > gpurun_out/pytest_r02c.log 2>&1
echo "pytest rc=$?"
tail -5 gpurun_out/pytest_r02c.log
for ta in 0 1; do python tools/run_pass.py --config c3 --ta $ta --reps 5; done > gpurun_out/pass_r02c.txt 2>&1
python tools/profile_stages.py --config c3 --reps 2 > gpurun_out/stages_c3_r02c.txt 2>&1
python tools/profile_stages.py --config c2 --reps 3 > gpurun_out/stages_c2_r02c.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_r02c.csv python tools/profile_stages.py --config c3 --reps 1 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "c3_full_fp64 or c4_full or c5_16384" > gpurun_out/pytest_full_r02c.log 2>&1
echo "pytest full rc=$?"
echo done
