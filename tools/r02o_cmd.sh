out=gpurun_out/r02o; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x > $out/pytest_dist.log 2>&1; echo "pytest exit $?" >> $out/pytest_dist.log
tail -25 $out/pytest_dist.log
