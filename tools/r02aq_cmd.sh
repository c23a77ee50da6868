out=gpurun_out/r02aq; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q -k "blocked or not panel" > $out/pytest.log 2>&1; echo "pytest exit $?"; tail -2 $out/pytest.log
for c in n5000_k16 n5000_k4 n5000_k64; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e > $out/b_$c.json 2>$out/b_$c.err
  python -c "import json; d=json.load(open('$out/b_$c.json')); print('$c', d['ms_per_step'], d['roofline']['frac'])"
done
GCM_LIB_PATH=paper_1011_1173_b200/lib/variants/libgcm_trace.so python tools/trace_chain.py 5000 16 2>&1 | tail -9
