# n=5000/8000 persistent chain: solver span (PC trace build) vs whole call, tail overlapped / not
for nk in "5000 16" "8000 16" "5000 32"; do
echo "== $nk"; GCM_LIB_PATH=$PWD/paper_1011_1173_b200/lib/variants/libgcm_pctrace.so timeout 120 python tools/pchain_trace.py $nk 2>&1 | tail -12
done
python - <<'PY'
import torch, sys, os
sys.path.insert(0,'.')
import paper_1011_1173_b200 as gcm
for n,k in [(5000,16),(8000,16)]:
    g=torch.Generator(device='cuda'); g.manual_seed(1)
    L=torch.empty((n,n),dtype=torch.float64,device='cuda'); L.uniform_(-1/n**0.5,1/n**0.5,generator=g); L.diagonal().uniform_(1.0,2.0,generator=g)
    V=torch.rand((k,n),dtype=torch.float64,device='cuda',generator=g)/n**0.5
    for tail in ['1','0']:
      for ch in ['8','4','2']:
        os.environ['GCM_PCHAIN_TAIL']=tail; os.environ['GCM_PCHAIN_CHUNKS']=ch
        ts=[]
        for i in range(6):
            Vc=V.clone(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
            e0.record(); gcm.modify(L,Vc,1 if i%2==0 else -1,algo='panel'); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        print(n,k,'tail',tail,'chunks',ch,[round(x,4) for x in sorted(ts)[:3]], flush=True)
        if tail=='0': break
PY
