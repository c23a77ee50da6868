timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k "panel or pchain or launch_chain or dist" 2>&1 | tail -2
for tail in 1 0; do for n in 5000 12000; do GCM_PCHAIN_TAIL=$tail python tools/scope_time.py $n 16 panel; done; GCM_PCHAIN_TAIL=$tail python tools/scope_time.py 20000 32 panel; done
for r in 16 32; do GCM_PCHAIN_RESERVE=$r python tools/scope_time.py 12000 16 panel; GCM_PCHAIN_RESERVE=$r python tools/scope_time.py 20000 32 panel; done
python tools/scope_time.py 5000 16 blocked
