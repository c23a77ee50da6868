timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02b_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02b_pytest.log
tail -3 gpurun_out/r02b_pytest.log
bash tools/r02_ncu.sh r02b
cat gpurun_out/r02b/rc.txt
