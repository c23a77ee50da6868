out=gpurun_out/r02t; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_edge.py tests/test_gpu_parity.py -q -x -k "panel or virtual or dist" > $out/pytest.log 2>&1; echo "pytest exit $?" >> $out/pytest.log
tail -3 $out/pytest.log
for c in n5000_k16 n100000_k32; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e --algo panel > $out/bench_${c}_panel.json 2> $out/bench_${c}_panel.err
python -c "import json; d=json.load(open('$out/bench_${c}_panel.json')); print('panel $c', d['ms_per_step'], d['kernels'], d.get('check'))"
done
