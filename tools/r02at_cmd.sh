out=gpurun_out/r02at; mkdir -p $out
python tools/panel_trace.py 40000 32 > $out/plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:pupdate_mma_kernel -s 11 -c 1 -o $out/pupdate -f python tools/panel_trace.py 40000 32 > $out/ncu.log 2>&1
echo rc=$?
