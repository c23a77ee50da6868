GCM_LIB_PATH=paper_1011_1173_b200/lib/variants/libgcm_skew.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_batched.py -q -x 2>&1 | tail -1
bash tools/ab.sh "base noskew skew" "n5000_k16 n5000_k64 batched n100000_k32" 2
