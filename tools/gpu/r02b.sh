set -x
python tools/dbg_jacobi_nan.py 150 200 256 > gpurun_out/dbg_jacobi_nan.txt 2>&1
timeout 300 compute-sanitizer --tool memcheck python tools/dbg_jacobi_nan.py 200 > gpurun_out/dbg_jacobi_nan_memcheck.txt 2>&1
for ta in 0 1; do python tools/run_pass.py --config c3 --ta $ta --reps 5; done > gpurun_out/pass_c3_r02b.txt 2>&1
python tools/run_pass.py --config c2 --ta 0 --reps 10 >> gpurun_out/pass_c3_r02b.txt 2>&1
python tools/profile_stages.py --config c3 --reps 2 > gpurun_out/stages_c3_r02b.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_r02b.csv python tools/profile_stages.py --config c3 --reps 1 > gpurun_out/ncu_launch_c3.log 2>&1
echo done
