out=gpurun_out/r02h; mkdir -p $out
V=$PWD/paper_1011_1173_b200/lib/variants
for bsz in 160 4096; do for v in bttrace2 bttrace3; do GCM_LIB_PATH=$V/libgcm_$v.so timeout 300 python tools/batched_trace.py $bsz > $out/trace_${v}_$bsz.txt 2>&1; done; done
grep -H total $out/trace_*.txt
