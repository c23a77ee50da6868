timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k "panel or pchain or launch_chain or dist" 2>&1 | tail -1
for a in "5000 16 panel" "10000 32 panel"; do python tools/host_overhead.py $a 2>&1 | tail -1; done
python tools/kernel_timeline.py 5000 16 panel -v 2>&1 | grep -E "pinv|pinit|pchain_kernel" | head -4
