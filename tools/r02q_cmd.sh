out=gpurun_out/r02q; mkdir -p $out
cmd="python bench.py --config n5000_k16 --steps 1 --warmup 3 --no-cpu --no-e2e --algo panel"
$cmd > $out/plain.json 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv $cmd > $out/ncu.log 2>&1
python tools/launches.py $out/launches.csv
