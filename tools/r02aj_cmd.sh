out=gpurun_out/r02aj; mkdir -p $out
python tools/panel_trace.py 20000 32 > $out/plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:pupdate -s 11 -c 1 -o $out/pupdate -f python tools/panel_trace.py 20000 32 > $out/ncu.log 2>&1
echo rc=$?
