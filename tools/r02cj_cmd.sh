timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k "panel or pchain or launch_chain or dist" 2>&1 | tail -1
python tools/kernel_timeline.py 5000 16 panel 2>&1 | grep -v -i warn | head -12
for v in base new base new; do
if [ $v = new ]; then unset GCM_LIB_PATH; else export GCM_LIB_PATH=$PWD/paper_1011_1173_b200/lib/variants/libgcm_$v.so; fi
for a in "5000 16 panel" "10000 32 panel"; do echo -n "$v "; python tools/host_overhead.py $a 2>&1 | tail -1; done
done
