timeout 900 python -m pytest tests/test_gpu_batched.py -q -x 2>&1 | tail -1
for w in 1 0; do GCM_BATCHED_W=$w timeout 900 python bench.py --config batched --steps 10 --warmup 3 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('batched W=$w', d['ms_per_step'], d['kernels'], d['roofline']['frac'])"; done
