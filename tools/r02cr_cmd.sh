out=gpurun_out/r02cr; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest exit $?"; tail -2 $out/pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for c in n5000_k16 n5000_k1 n5000_k4 n5000_k64 batched n100000_k32; do
  timeout 600 python bench.py --config $c > $out/b_$c.json 2>$out/b_$c.err
  python -c "import json; d=json.load(open('$out/b_$c.json')); print('$c', d['ms_per_step'], d['value'], d['unit'], 'frac', d['roofline']['frac'], d['roofline']['kernel'], 'e2e', d['e2e']['value'] if d.get('e2e') else None, 'launches', d.get('gpu_launches'))" 2>&1 | tail -1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_n5000_k16.csv python bench.py --steps 2 --warmup 3 > $out/ncu.log 2>&1; echo "ncu exit $?"
