cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/a
GCM_LIB_PATH=paper_1011_1173_b200/lib/variants/libgcm_sw5.so timeout 120 python tools/trace_bdiag.py 5000 16 > gpurun_out/a/tb.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/a/pytest.txt 2>&1
