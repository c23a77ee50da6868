timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -k "launch_chain or pchain or virtual" 2>&1 | tail -1
for gq in 8 4 16; do GCM_LC_GROUPS=$gq timeout 900 python bench.py --config n100000_k32 --steps 3 --warmup 3 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n1e5 groups=$gq', d['ms_per_step'], d['check']['ok'])"; done
GCM_LC_OVERLAP=0 timeout 900 python bench.py --config n100000_k32 --steps 3 --warmup 3 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n1e5 no overlap', d['ms_per_step'])"
