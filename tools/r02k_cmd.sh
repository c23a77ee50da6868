out=gpurun_out/r02k; mkdir -p $out
V=$PWD/paper_1011_1173_b200/lib/variants
for rep in 1 2; do for v in b_m2_s2 b_m2_s3 b_m3_s2 b_m3_s3; do
  GCM_LIB_PATH=$V/libgcm_$v.so timeout 300 python bench.py --config batched --steps 10 --warmup 3 --no-cpu --no-e2e > $out/bench_$v.json 2>&1
  python -c "import json; d=json.load(open('$out/bench_$v.json')); print('$v', d['ms_per_step'], d['roofline']['frac'])"
done; done
