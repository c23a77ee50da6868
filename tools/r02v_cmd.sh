out=gpurun_out/r02v; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_f32.py -q -x > $out/pytest.log 2>&1; echo "pytest exit $?" >> $out/pytest.log
tail -15 $out/pytest.log
timeout 1500 python tools/paper_grid.py --out $out/paper_grid > $out/grid.log 2>&1; echo grid rc=$?
tail -5 $out/grid.log
