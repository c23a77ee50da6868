timeout 900 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k panel 2>&1 | tail -2
python - <<'PY'
import torch, sys, os
sys.path.insert(0,'.')
import paper_1011_1173_b200 as gcm
for n,k in [(5000,16),(12000,16),(20000,32),(40000,32)]:
    g=torch.Generator(device='cuda'); g.manual_seed(1)
    L=torch.empty((n,n),dtype=torch.float64,device='cuda'); L.uniform_(-1/n**0.5,1/n**0.5,generator=g); L.diagonal().uniform_(1.0,2.0,generator=g)
    V=torch.rand((k,n),dtype=torch.float64,device='cuda',generator=g)/n**0.5
    for algo in ['blocked','panel']:
        for pc in (['1','0'] if algo=='panel' else ['1']):
            os.environ['GCM_PCHAIN']=pc
            ts=[]
            for i in range(6):
                Vc=V.clone(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
                e0.record(); gcm.modify(L,Vc,1 if i%2==0 else -1,algo=algo); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
            print(n,k,algo,'pchain',pc,'ms',[round(x,4) for x in sorted(ts)[:3]], flush=True)
    del L, V; torch.cuda.empty_cache()
os.environ['GCM_PCHAIN']='1'
PY
for v in 1 0; do GCM_PCHAIN=$v timeout 900 python bench.py --config n100000_k32 --steps 3 --warmup 3 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n1e5 pchain=$v', d['ms_per_step'], d['kernels'], d['check']['ok'])"; done
GCM_LIB_PATH=paper_1011_1173_b200/lib/variants/libgcm_pctrace.so python tools/pchain_trace.py 5000 16
