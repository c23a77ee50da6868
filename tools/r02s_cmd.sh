out=gpurun_out/r02s; mkdir -p $out
cmd="python bench.py --config n5000_k16 --steps 1 --warmup 3 --no-cpu --no-e2e --algo panel"
$cmd > $out/plain.json 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:dsolve -s 35 -c 1 -o $out/dsolve -f $cmd > $out/ncu.log 2>&1
echo rc=$?
