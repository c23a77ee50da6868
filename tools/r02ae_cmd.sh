out=gpurun_out/r02ae; mkdir -p $out
python /tmp/pu.py > $out/plain.log 2>&1 || { cp tools/r02ad_cmd.sh /tmp/x.sh; bash /tmp/x.sh > /dev/null 2>&1; }
python /tmp/pu.py > $out/plain.log 2>&1 && timeout 600 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --warp-sampling-interval 0 --import-source on --clock-control none -k regex:dsolve -s 100 -c 1 -o $out/dsolve -f python /tmp/pu.py > $out/ncu.log 2>&1
echo rc=$?
