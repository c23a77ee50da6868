out=gpurun_out/r02c; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_batched.py tests/test_gpu_edge.py -q -x > $out/pytest.log 2>&1; echo "pytest exit $?" >> $out/pytest.log
timeout 300 python bench.py --config batched --steps 10 --warmup 3 --no-cpu > $out/bench_batched.json 2> $out/bench_batched.err
GCM_BATCHED_LEGACY=1 timeout 300 python bench.py --config batched --steps 10 --warmup 3 --no-cpu > $out/bench_batched_legacy.json 2>&1
tail -3 $out/pytest.log; python -c "
import json
for f in ['bench_batched','bench_batched_legacy']:
    try:
        d=json.load(open('$out/'+f+'.json')); print(f, d['ms_per_step'], d['roofline']['frac'], d['roofline']['achieved'])
    except Exception as e: print(f, 'ERR', e)
"
cat $out/bench_batched.err | tail -5
