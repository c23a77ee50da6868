#!/bin/bash
# One GPU-box pass: GPU tests, bench lines, launch list and one ncu --set full capture.
# Usage (from the repo root on the box): bash tools/gpu_check.sh [tag]
tag=${1:-chk}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest exit $?" >> $out/pytest.log
for c in n5000_k16 n5000_k1 n5000_k4 n5000_k64 batched; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 4 > $out/bench_$c.json 2> $out/bench_$c.err
done
timeout 600 python bench.py --config n100000_k32 --steps 3 --warmup 3 > $out/bench_n100000_k32.json 2> $out/bench_n100000_k32.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > $out/bench_reference.json 2> $out/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'trsv|btma|bdiag' -s 6 -c 3 \
  -o $out/full -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $out/ncu_full.log 2>&1
echo done > $out/DONE
