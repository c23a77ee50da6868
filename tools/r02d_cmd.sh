out=gpurun_out/r02d; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_batched.py tests/test_gpu_edge.py -q -x > $out/pytest.log 2>&1; echo "pytest exit $?" >> $out/pytest.log
tail -2 $out/pytest.log
cmd="python bench.py --config batched --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 300 $cmd > $out/bench_batched.json 2> $out/bench_batched.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batched -s 3 -c 1 -o $out/full_batched -f $cmd > $out/ncu.log 2>&1
echo "ncu rc=$?"
python -c "
import json; d=json.load(open('$out/bench_batched.json')); print(d['ms_per_step'], d['roofline']['frac'])"
