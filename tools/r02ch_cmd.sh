for a in "5000 16 panel" "5000 16 blocked" "10000 32 panel" "5000 64 blocked"; do python tools/host_overhead.py $a 2>&1 | tail -1; done
