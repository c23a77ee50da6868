out=gpurun_out/r02bg; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest exit $?"; tail -2 $out/pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for c in n5000_k16 n5000_k1 n5000_k4 n5000_k64 batched n100000_k32 n100000_k32_dist; do
  timeout 900 python bench.py --config $c > $out/b_$c.json 2>$out/b_$c.err
  python -c "import json; d=json.load(open('$out/b_$c.json')); print('$c', d['ms_per_step'], d['value'], d['unit'], 'frac', d['roofline']['frac'], d['roofline']['kernel'], 'e2e', d['e2e']['value'] if d.get('e2e') else None)" 2>&1 | tail -1
done
python - <<'PY' > gpurun_out/r02bg/crossover.txt 2>&1
import torch, sys, os
sys.path.insert(0,'.')
import paper_1011_1173_b200 as gcm
print("# n, k, algo (panel: GCM_PCHAIN=1 persistent chain / 0 per-solve-block launches), best-3 ms of 6 alternating update/downdate calls, B200")
for n,k in [(8000,16),(12000,16),(12000,32),(16000,16),(16000,32),(20000,16),(20000,32),(40000,32)]:
    g=torch.Generator(device='cuda'); g.manual_seed(1)
    L=torch.empty((n,n),dtype=torch.float64,device='cuda'); L.uniform_(-1/n**0.5,1/n**0.5,generator=g); L.diagonal().uniform_(1.0,2.0,generator=g)
    V=torch.rand((k,n),dtype=torch.float64,device='cuda',generator=g)/n**0.5
    for algo, pc in [('blocked','1'),('panel','1'),('panel','0')]:
        os.environ['GCM_PCHAIN']=pc
        ts=[]
        for i in range(6):
            Vc=V.clone(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
            e0.record(); gcm.modify(L,Vc,1 if i%2==0 else -1,algo=algo); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        print(n,k,algo,'pchain='+pc,[round(x,4) for x in sorted(ts)[:3]], flush=True)
    del L, V; torch.cuda.empty_cache()
PY
cat gpurun_out/r02bg/crossover.txt
