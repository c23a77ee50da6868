#!/bin/bash
# One GPU-box pass for round 2: FP64 peak + link latencies, the GPU suite, the near-singular
# error levels, and the headline bench line.  Usage (repo root on the box): bash tools/r02_check.sh TAG
tag=${1:-r02}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > $out/fp64_peak.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q --durations=15 > $out/pytest.log 2>&1; echo "pytest exit $?" >> $out/pytest.log
timeout 300 python tools/near_singular_probe.py > $out/near_singular.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 4 > $out/bench_n5000_k16.json 2> $out/bench_n5000_k16.err
echo done > $out/DONE
