out=gpurun_out/r02e; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_edge.py tests/test_gpu_batched.py tests/test_gpu_parity.py -q -x > $out/pytest.log 2>&1; echo "pytest exit $?" >> $out/pytest.log
tail -2 $out/pytest.log
GCM_LIB_PATH=$PWD/paper_1011_1173_b200/lib/variants/libgcm_bttrace.so timeout 300 python tools/batched_trace.py > $out/bt_trace.txt 2>&1
cat $out/bt_trace.txt
