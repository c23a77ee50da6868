# chaos build (random pauses before every publish and poll) on the panel / persistent-chain tests
out=gpurun_out/r02ct; mkdir -p $out
GCM_LIB_PATH=$PWD/paper_1011_1173_b200/lib/variants/libgcm_chaos.so timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -p no:cacheprovider -k "panel or pchain or launch_chain or dist or large_n or headline" > $out/pytest.log 2>&1
echo "chaos pytest rc=$?"; tail -1 $out/pytest.log
