timeout 900 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k panel 2>&1 | tail -1
for v in 1 0; do GCM_PCHAIN=$v timeout 900 python bench.py --config n100000_k32 --steps 3 --warmup 3 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n1e5 pchain=$v', d['ms_per_step'], d['kernels'], d['check'])"; done
