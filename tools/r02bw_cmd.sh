timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x 2>&1 | tail -1
bash tools/ab.sh "pair1 pair0" "n5000_k16 n5000_k4 n5000_k64" 3
