timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ozaki.py tests/test_gpu_multirank.py -q -rf -p no:cacheprovider -k "k512 or thin_qr or qr or config5 or big or multirank or sharded" > gpurun_out/pytest_r02k.log 2>&1
echo "rc=$?"; tail -15 gpurun_out/pytest_r02k.log
python tools/profile_stages.py --config c5 --reps 1 > gpurun_out/stages_c5_r02k.txt 2>&1
