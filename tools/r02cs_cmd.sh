# DRAM bytes per kernel of the persistent-chain path (n5000_k16 and k4/k1), for the pchain scope's traffic
out=gpurun_out/r02cs; mkdir -p $out
for c in n5000_k16 n5000_k4 n5000_k1; do
cmd="python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 300 $cmd > $out/plain_$c.json 2>$out/plain_$c.err && \
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $out/dram_$c.csv $cmd > $out/ncu_$c.log 2>&1
echo "$c rc=$?"
done
