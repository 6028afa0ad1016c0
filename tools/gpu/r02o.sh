timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_ozaki.py -q -rf -p no:cacheprovider > gpurun_out/pytest_r02o.log 2>&1
echo "rc=$?"; tail -5 gpurun_out/pytest_r02o.log
