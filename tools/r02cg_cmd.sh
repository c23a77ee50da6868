python tools/kernel_timeline.py 5000 16 panel -v 2>&1 | grep -v Warning | head -80
python tools/kernel_timeline.py 5000 16 blocked 2>&1 | grep -v Warning | head -20
