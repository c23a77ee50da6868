out=gpurun_out/r02f; mkdir -p $out
V=$PWD/paper_1011_1173_b200/lib/variants
for v in bttrace3 bttrace2; do GCM_LIB_PATH=$V/libgcm_$v.so timeout 300 python tools/batched_trace.py > $out/trace_$v.txt 2>&1; done
for v in default bt2; do
  if [ $v = default ]; then unset GCM_LIB_PATH; else export GCM_LIB_PATH=$V/libgcm_$v.so; fi
  timeout 300 python bench.py --config batched --steps 10 --warmup 3 --no-cpu --no-e2e > $out/bench_$v.json 2>&1
  python -c "import json; d=json.load(open('$out/bench_$v.json')); print('$v', d['ms_per_step'], d['roofline']['frac'])"
done
unset GCM_LIB_PATH
grep total $out/trace_*.txt
