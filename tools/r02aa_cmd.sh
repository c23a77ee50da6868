out=gpurun_out/r02aa; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -x > $out/pytest.log 2>&1; echo "pytest exit $?" >> $out/pytest.log
tail -3 $out/pytest.log
for c in n5000_k16 n5000_k4 batched; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 4 --no-cpu --no-e2e > $out/bench_$c.json 2>&1
  python -c "import json; d=json.load(open('$out/bench_$c.json')); print('$c', d['ms_per_step'], d['roofline']['frac'], d['roofline_path']['frac'] if 'roofline_path' in d else '')"
done
