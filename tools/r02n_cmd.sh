out=gpurun_out/r02n; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $out/pytest.log 2>&1; echo "pytest exit $?" >> $out/pytest.log
tail -14 $out/pytest.log
timeout 300 python bench.py --config batched --steps 20 --warmup 4 --no-cpu > $out/bench_batched.json 2> $out/bench_batched.err
python -c "import json; d=json.load(open('$out/bench_batched.json')); print('batched', d['ms_per_step'], d['roofline']['frac'], d['roofline']['achieved'])"
