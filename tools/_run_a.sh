cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/a
timeout 60 python tools/quick_time.py 5000 16 > gpurun_out/a/qt.txt 2>&1 || { echo "quick_time failed $?" >> gpurun_out/a/qt.txt; exit 0; }
timeout 60 python tools/quick_time.py 5000 4 >> gpurun_out/a/qt.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/a/pytest.txt 2>&1
for c in n5000_k16 n5000_k1 n5000_k4 n5000_k64; do timeout 120 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/a/bench_$c.json 2>&1; done
GCM_LIB_PATH=paper_1011_1173_b200/lib/variants/libgcm_cur.so timeout 60 python tools/trace_chain.py 5000 16 > gpurun_out/a/tc.txt 2>&1
