out=gpurun_out/r02ab; mkdir -p $out
GCM_LIB_PATH=$PWD/paper_1011_1173_b200/lib/variants/libgcm_trace.so python tools/trace_helper.py 5000 16 2>&1 | head -6
GCM_LIB_PATH=$PWD/paper_1011_1173_b200/lib/variants/libgcm_trace.so python tools/trace_chain.py 5000 16 2>&1 | sed -n 10,14p
for rep in 1 2; do for v in new base; do
  if [ $v = new ]; then unset GCM_LIB_PATH; else export GCM_LIB_PATH=$PWD/paper_1011_1173_b200/lib/variants/libgcm_$v.so; fi
  for c in n5000_k16 n5000_k4 n5000_k64; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 4 --no-cpu --no-e2e > $out/b_${c}_$v.json 2>&1
  python -c "import json; d=json.load(open('$out/b_${c}_$v.json')); print('$v $c', d['ms_per_step'])"
  done
done; done
unset GCM_LIB_PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x 2>&1 | tail -2
