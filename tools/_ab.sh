cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
timeout 120 python tools/quick_time.py 5000 16 > gpurun_out/ab/qt.txt 2>&1 || { echo "quick_time failed" >> gpurun_out/ab/qt.txt; exit 0; }

for rep in 1 2; do for v in pdl2 pub3 pub7; do for c in n5000_k16 n5000_k4 n5000_k1; do
GCM_LIB_PATH=paper_1011_1173_b200/lib/variants/libgcm_$v.so timeout 120 python bench.py --config $c --steps 20 --warmup 4 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c', d['ms_per_step'], {k:round(v['ms_total']/v['launches']*1000,1) for k,v in d['kernels'].items()})"
done; done; done > gpurun_out/ab/ab.txt 2>&1
