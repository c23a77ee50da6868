out=gpurun_out/r02g; mkdir -p $out
V=$PWD/paper_1011_1173_b200/lib/variants
for v in bttr_rg2 bttr_rg4 bttr_rg8; do GCM_LIB_PATH=$V/libgcm_$v.so timeout 300 python tools/batched_trace.py > $out/trace_$v.txt 2>&1; done
grep -H total $out/trace_*.txt
