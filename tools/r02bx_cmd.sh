timeout 900 python -m pytest tests/test_gpu_batched.py -q -x 2>&1 | tail -1
GCM_BT_CFG=192 timeout 900 python -m pytest tests/test_gpu_batched.py -q -x 2>&1 | tail -1
for rep in 1 2; do for c in 256 192; do GCM_BT_CFG=$c timeout 900 python bench.py --config batched --steps 10 --warmup 3 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('batched cfg=$c', d['ms_per_step'], d['roofline']['frac'])"; done; done
