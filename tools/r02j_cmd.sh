out=gpurun_out/r02j; mkdir -p $out
V=$PWD/paper_1011_1173_b200/lib/variants
GCM_LIB_PATH=$V/libgcm_bttr.so timeout 300 python tools/batched_trace.py > $out/trace.txt 2>&1
cat $out/trace.txt | tail -22
timeout 300 python bench.py --config batched --steps 10 --warmup 3 --no-cpu --no-e2e > $out/bench.json 2>&1
python -c "import json; d=json.load(open('$out/bench.json')); print(d['ms_per_step'], d['roofline']['frac'])"
timeout 600 python -m pytest tests/test_gpu_batched.py tests/test_gpu_edge.py -q -x -k batched 2>&1 | tail -2
