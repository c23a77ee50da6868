out=gpurun_out/r02az; mkdir -p $out
python tools/panel_trace.py 20000 32 > $out/plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:papply -s 1 -c 1 -o $out/papply -f python tools/panel_trace.py 20000 32 > $out/ncu.log 2>&1
echo rc=$?
