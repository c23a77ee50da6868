timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k "panel or pchain or launch_chain or dist" 2>&1 | tail -2
for s in 1 0; do GCM_APPLY_SPLIT=$s python tools/scope_time.py 20000 32 panel; GCM_APPLY_SPLIT=$s python tools/scope_time.py 12000 16 panel; done
for s in 1 0; do GCM_APPLY_SPLIT=$s timeout 900 python bench.py --config n100000_k32 --steps 3 --warmup 3 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n1e5 split=$s', d['ms_per_step'], d['kernels'], d['check']['ok'])"; done
