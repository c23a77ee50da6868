timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k "not panel" 2>&1 | tail -1
bash tools/ab.sh "base pf" "n5000_k16 n5000_k64 n5000_k4" 3
