out=gpurun_out/r02m; mkdir -p $out
V=$PWD/paper_1011_1173_b200/lib/variants
for rep in 1 2; do for v in A B C D E; do
  GCM_LIB_PATH=$V/libgcm_$v.so timeout 300 python bench.py --config batched --steps 10 --warmup 3 --no-cpu --no-e2e > $out/bench_$v.json 2>&1
  python -c "import json; d=json.load(open('$out/bench_$v.json')); print('$v', d['ms_per_step'], d['roofline']['frac'])"
done; done
