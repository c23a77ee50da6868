#!/bin/bash
# Same-box A/B of library variants (tools/build_variant.sh NAME -D... builds
# paper_1011_1173_b200/lib/variants/libgcm_NAME.so). Run on the GPU box, e.g.
#   gpurun -- 'bash tools/ab.sh "old new" "n5000_k16 n5000_k4" 2'
# Prints one line per (rep, variant, config): ms/step and the per-scope kernel times.
variants=${1:-"new"}; configs=${2:-"n5000_k16"}; reps=${3:-2}
mkdir -p gpurun_out/ab
for rep in $(seq $reps); do for v in $variants; do for c in $configs; do
  GCM_LIB_PATH=paper_1011_1173_b200/lib/variants/libgcm_$v.so timeout 300 python bench.py --config $c --steps 20 \
    --warmup 4 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c', d['ms_per_step'], {k:round(v['ms_total']/v['launches']*1000,1) for k,v in d['kernels'].items()})"
done; done; done | tee gpurun_out/ab/ab.txt
