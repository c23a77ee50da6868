# knob sweep on the final build: tail chunks (GCM_PCHAIN_CHUNKS) and helper rowcnt release batch (GCM_PC_REL variants)
for v in new rel2 rel8; do for ch in 8 6 4; do
if [ $v = new ]; then unset GCM_LIB_PATH; else export GCM_LIB_PATH=$PWD/paper_1011_1173_b200/lib/variants/libgcm_$v.so; fi
if [ $v != new ] && [ $ch != 8 ]; then continue; fi
GCM_PCHAIN_CHUNKS=$ch V=$v timeout 300 python - <<'PY'
import torch, sys, os
sys.path.insert(0,'.')
import paper_1011_1173_b200 as gcm
out=[]
for n,k in [(5000,16),(8000,16),(10000,32)]:
    g=torch.Generator(device='cuda'); g.manual_seed(1)
    L=torch.empty((n,n),dtype=torch.float64,device='cuda'); L.uniform_(-1/n**0.5,1/n**0.5,generator=g); L.diagonal().uniform_(1.0,2.0,generator=g)
    V=torch.rand((k,n),dtype=torch.float64,device='cuda',generator=g)/n**0.5
    Vc=V.clone(); ts=[]
    for i in range(12):
        Vc.copy_(V); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); gcm.modify(L,Vc,1 if i%2==0 else -1,algo='panel'); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    out.append(f"{n}/{k} {sorted(ts)[1]:.4f}")
    del L,V,Vc; torch.cuda.empty_cache()
print(os.environ['V'], 'chunks', os.environ['GCM_PCHAIN_CHUNKS'], ' '.join(out), flush=True)
PY
done; done
