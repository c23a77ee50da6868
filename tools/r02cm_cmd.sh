timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k "panel or pchain or launch_chain or dist" 2>&1 | tail -1
GCM_TAIL_GRAPH=0 timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -k "pchain" 2>&1 | tail -1
for g in 1 0 1 0; do for a in "5000 16 panel" "10000 32 panel"; do echo -n "graph=$g "; GCM_TAIL_GRAPH=$g GCM_HOST_TRACE=1 python tools/host_overhead.py $a 2>&1 | grep -E "host_trace|host enq" | tail -2 | tr '\n' ' '; echo; done; done
