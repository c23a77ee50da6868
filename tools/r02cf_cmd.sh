# solver hand-off poller warps: parity (panel/pchain tests), then base vs new timing, then trace
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k "panel or pchain or launch_chain or dist" 2>&1 | tail -2
GCM_LIB_PATH=$PWD/paper_1011_1173_b200/lib/variants/libgcm_pctrace.so timeout 120 python tools/pchain_trace.py 5000 16 2>&1 | tail -12
for v in base new base new; do
if [ $v = new ]; then unset GCM_LIB_PATH; else export GCM_LIB_PATH=$PWD/paper_1011_1173_b200/lib/variants/libgcm_$v.so; fi
V=$v python - <<'PY'
import torch, sys, os
sys.path.insert(0,'.')
import paper_1011_1173_b200 as gcm
out=[]
for n,k in [(5000,16),(7000,16),(10000,32),(20000,32)]:
    g=torch.Generator(device='cuda'); g.manual_seed(1)
    L=torch.empty((n,n),dtype=torch.float64,device='cuda'); L.uniform_(-1/n**0.5,1/n**0.5,generator=g); L.diagonal().uniform_(1.0,2.0,generator=g)
    V=torch.rand((k,n),dtype=torch.float64,device='cuda',generator=g)/n**0.5
    ts=[]
    for i in range(8):
        Vc=V.clone(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); gcm.modify(L,Vc,1 if i%2==0 else -1,algo='panel'); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    out.append(f"{n}/{k} {sorted(ts)[1]:.4f}")
    del L,V; torch.cuda.empty_cache()
print(os.environ['V'], ' '.join(out), flush=True)
PY
done
