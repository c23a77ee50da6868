out=gpurun_out/r02ap; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest exit $?"; tail -3 $out/pytest.log
for c in n5000_k16 n5000_k4 n5000_k64 n5000_k1; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e > $out/b_$c.json 2>$out/b_$c.err
  python -c "import json; d=json.load(open('$out/b_$c.json')); print('$c', d['ms_per_step'], d['roofline']['frac'])"
done
bash tools/build_variant.sh trace -DGCM_TRACE > /dev/null 2>&1
GCM_LIB_PATH=paper_1011_1173_b200/lib/variants/libgcm_trace.so python tools/trace_chain.py 5000 16 2>&1 | sed -n '1,30p'
GCM_LIB_PATH=paper_1011_1173_b200/lib/variants/libgcm_trace.so python tools/trace_helper.py 5000 16 2>&1 | head -6
