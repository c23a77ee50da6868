out=gpurun_out/r02w; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x > $out/pytest.log 2>&1; echo "pytest exit $?" >> $out/pytest.log
tail -3 $out/pytest.log
for rep in 1 2; do
for v in closed wave; do
  if [ $v = closed ]; then unset GCM_LIB_PATH; else export GCM_LIB_PATH=$PWD/paper_1011_1173_b200/lib/variants/libgcm_$v.so; fi
  for c in n5000_k16 n5000_k4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 4 --no-cpu --no-e2e > $out/bench_${c}_$v.json 2>&1
  python -c "import json; d=json.load(open('$out/bench_${c}_$v.json')); print('$v $c', d['ms_per_step'], d['roofline_path']['frac'])"
  done
done; done
unset GCM_LIB_PATH
