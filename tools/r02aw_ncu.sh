#!/bin/bash
# Per-config ncu evidence (one gpurun call = one ncu "use"): for every bench config, the plain
# run first (must exit 0), then `ncu --set full` on the dominant kernels after the warm-up
# launches, then a launch list.  n100000_k32 (80 GB factor: kernel replay would save/restore it)
# gets application replay of the DRAM-byte and duration metrics only.
# Usage (repo root on the box): bash tools/r02aw_ncu.sh TAG   (round 2, after the DMMA panel path:
# n100000_k32's dominant kernel is papply)
tag=${1:-r02aw}
out=gpurun_out/$tag
mkdir -p $out
run() {  # config skip-launches count
  c=$1; s=$2; n=$3
  cmd="python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu"
  timeout 600 $cmd > $out/plain_$c.json 2> $out/plain_$c.err &&
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'trsv|btma|btile|bapply|batched' \
      -s $s -c $n -o $out/full_$c -f $cmd > $out/ncu_$c.log 2>&1
  echo "$c ncu rc=$?" >> $out/rc.txt
}
run n5000_k16 6 2
run n5000_k1 6 2
run n5000_k4 6 2
run n5000_k64 12 4
run batched 3 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_n5000_k16.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $out/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 50 --csv --log-file $out/launches_batched.csv \
  python bench.py --config batched --steps 2 --warmup 3 --no-e2e --no-cpu > $out/ncu_launch_b.log 2>&1
c=n100000_k32
cmd="python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 900 $cmd > $out/plain_$c.json 2> $out/plain_$c.err &&
timeout 1500 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:'papply' -s 3 -c 1 --csv --log-file $out/app_$c.csv $cmd > $out/ncu_$c.log 2>&1
echo "$c papply ncu rc=$?" >> $out/rc.txt
timeout 1500 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:'dsolve|pupdate_mma_kernel<32>' -s 2400 -c 2 --csv --log-file $out/app2_$c.csv $cmd > $out/ncu2_$c.log 2>&1
echo "$c chain ncu rc=$?" >> $out/rc.txt
echo done > $out/DONE
