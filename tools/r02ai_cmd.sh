out=gpurun_out/r02ai; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k panel 2>&1 | tail -2
bash tools/r02ad_cmd.sh 2>&1 | grep "dsolve\|pupdate\|lookahead\|pinv"
timeout 900 python bench.py --config n100000_k32 --steps 3 --warmup 3 --no-cpu --no-e2e > $out/b.json 2>&1
python -c "import json; d=json.load(open('$out/b.json')); print('n1e5 panel', d['ms_per_step'], d['kernels'])"
