out=gpurun_out/r02p; mkdir -p $out
for a in panel blocked; do
timeout 900 python bench.py --config n100000_k32 --steps 3 --warmup 3 --no-cpu --algo $a > $out/bench_n1e5_$a.json 2> $out/bench_n1e5_$a.err
python -c "import json; d=json.load(open('$out/bench_n1e5_$a.json')); print('$a n1e5', d['ms_per_step'], d['kernels'], d.get('check'))"
done
for a in panel blocked; do
timeout 300 python bench.py --config n5000_k16 --steps 10 --warmup 3 --no-cpu --no-e2e --algo $a > $out/bench_n5000_$a.json 2>&1
python -c "import json; d=json.load(open('$out/bench_n5000_$a.json')); print('$a n5000', d['ms_per_step'], d['kernels'])"
done
