for c in 2 3 4; do for n in 5000 12000; do GCM_PCHAIN_CHUNKS=$c python tools/scope_time.py $n 16 panel; done; GCM_PCHAIN_CHUNKS=$c python tools/scope_time.py 20000 32 panel; done
GCM_PCHAIN_CHUNKS=2 GCM_PCHAIN_RESERVE=24 python tools/scope_time.py 12000 16 panel
GCM_PCHAIN_CHUNKS=2 GCM_PCHAIN_RESERVE=24 python tools/scope_time.py 20000 32 panel
