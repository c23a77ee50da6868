cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
GCM_LIB_PATH=paper_1011_1173_b200/lib/variants/libgcm_f32p.so timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest.txt 2>&1
for rep in 1 2; do for v in old cur f32p; do for c in n5000_k64 n5000_k16; do
GCM_LIB_PATH=paper_1011_1173_b200/lib/variants/libgcm_$v.so timeout 120 python bench.py --config $c --steps 20 --warmup 4 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c', d['ms_per_step'], {k:round(v['ms_total']/v['launches']*1000,1) for k,v in d['kernels'].items()})"
done; done; done > gpurun_out/ab/ab.txt 2>&1
