out=gpurun_out/r02r; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_edge.py -q -x -k "panel or virtual or dist" > $out/pytest.log 2>&1; echo "pytest exit $?" >> $out/pytest.log
tail -3 $out/pytest.log
cmd="python bench.py --config n5000_k16 --steps 1 --warmup 3 --no-cpu --no-e2e --algo panel"
$cmd > $out/plain.json 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv $cmd > $out/ncu.log 2>&1
python tools/launches.py $out/launches.csv
timeout 900 python bench.py --config n100000_k32 --steps 3 --warmup 3 --no-cpu --algo panel > $out/bench_n1e5_panel.json 2> $out/bench_n1e5_panel.err
python -c "import json; d=json.load(open('$out/bench_n1e5_panel.json')); print('panel n1e5', d['ms_per_step'], d['kernels'], d.get('check'))"
