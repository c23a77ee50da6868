out=gpurun_out/r02an; mkdir -p $out
python tools/panel_trace.py 5000 16 2>&1 | tail -1
python tools/panel_trace.py 20000 16 2>&1 | tail -1
python - <<'PY'
import torch, time, sys
sys.path.insert(0,'.')
import paper_1011_1173_b200 as gcm
for n,k in [(5000,16),(20000,16),(20000,32)]:
    g=torch.Generator(device='cuda'); g.manual_seed(1)
    L=torch.empty((n,n),dtype=torch.float64,device='cuda'); L.uniform_(-1/n**0.5,1/n**0.5,generator=g); L.diagonal().uniform_(1.0,2.0,generator=g)
    V=torch.rand((k,n),dtype=torch.float64,device='cuda',generator=g)/n**0.5
    for algo in ['blocked','panel']:
        ts=[]
        for i in range(6):
            Vc=V.clone(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
            e0.record(); gcm.modify(L,Vc,1 if i%2==0 else -1,algo=algo); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        print(n,k,algo,'ms',sorted(ts)[:3])
PY
timeout 900 python bench.py --config n100000_k32 --steps 3 --warmup 3 --no-cpu --no-e2e > $out/b.json 2>&1
python -c "import json; d=json.load(open('$out/b.json')); print('n1e5 panel', d['ms_per_step'], d['kernels'], d['roofline'])"
