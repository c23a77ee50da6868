timeout 900 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -1
for c in 2 4 8; do for n in 5000 8000; do GCM_PCHAIN_CHUNKS=$c python tools/scope_time.py $n 16 panel; done; GCM_PCHAIN_CHUNKS=$c python tools/scope_time.py 12000 32 panel; done
python tools/scope_time.py 5000 16 blocked
