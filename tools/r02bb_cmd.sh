timeout 900 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k panel 2>&1 | tail -1
python tools/panel_trace.py 100000 32 2>&1 | tail -1
GCM_PU_WAVES=2 python tools/panel_trace.py 100000 32 2>&1 | tail -1
GCM_PU_WAVES=4 python tools/panel_trace.py 100000 32 2>&1 | tail -1
python tools/panel_trace.py 100000 16 2>&1 | tail -1
