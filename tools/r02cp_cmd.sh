out=gpurun_out/r02cp; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest exit $?"; tail -2 $out/pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for c in n5000_k16 n5000_k1 n5000_k4 n5000_k64 batched n100000_k32 n100000_k32_dist; do
  timeout 900 python bench.py --config $c > $out/b_$c.json 2>$out/b_$c.err
  python -c "import json; d=json.load(open('$out/b_$c.json')); print('$c', d['ms_per_step'], d['value'], d['unit'], 'frac', d['roofline']['frac'], d['roofline']['kernel'], 'e2e', d['e2e']['value'] if d.get('e2e') else None)" 2>&1 | tail -1
done
python - <<'PY'
import torch, sys, os
sys.path.insert(0,'.')
import paper_1011_1173_b200 as gcm
for n,k in [(4000,16),(5000,16),(6000,16),(5000,4),(5000,32),(7000,32),(10000,32)]:
    g=torch.Generator(device='cuda'); g.manual_seed(1)
    L=torch.empty((n,n),dtype=torch.float64,device='cuda'); L.uniform_(-1/n**0.5,1/n**0.5,generator=g); L.diagonal().uniform_(1.0,2.0,generator=g)
    V=torch.rand((k,n),dtype=torch.float64,device='cuda',generator=g)/n**0.5
    Vc=V.clone()
    for algo in ['blocked','panel']:
        ts=[]
        for i in range(10):
            Vc.copy_(V); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
            e0.record(); gcm.modify(L,Vc,1 if i%2==0 else -1,algo=algo); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        print('xover',n,k,algo,[round(x,4) for x in sorted(ts)[:3]], flush=True)
    del L, V, Vc; torch.cuda.empty_cache()
PY
