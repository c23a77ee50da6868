cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest.txt 2>&1
timeout 600 python bench.py --config n100000_k32 --steps 3 --warmup 3 > gpurun_out/ab/n1e5.json 2> gpurun_out/ab/n1e5.err
for c in n5000_k16 n5000_k1 n5000_k4 n5000_k64; do timeout 300 python bench.py --config $c --steps 20 --warmup 4 > gpurun_out/ab/bench_$c.json 2> gpurun_out/ab/bench_$c.err; done
