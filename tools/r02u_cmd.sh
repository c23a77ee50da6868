out=gpurun_out/r02u; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x > $out/pytest.log 2>&1; echo "pytest exit $?" >> $out/pytest.log
tail -3 $out/pytest.log
timeout 900 python bench.py --config n100000_k32_dist --steps 3 --warmup 3 --no-cpu > $out/bench_dist.json 2> $out/bench_dist.err
python -c "import json; d=json.load(open('$out/bench_dist.json')); print('dist N=1', d['ms_per_step'], d['value'], d['gpu_launches'], d['kernels'], d.get('check'), d['scaling'], d['roofline']['kernel'], d['roofline']['frac'])"
tail -3 $out/bench_dist.err
