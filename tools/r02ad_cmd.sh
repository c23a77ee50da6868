out=gpurun_out/r02ad; mkdir -p $out
python /tmp/pu.py > $out/plain.log 2>&1 || { cat > /tmp/pu.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_1011_1173_b200 as gcm
n, k = 20000, 32
g = torch.Generator(device='cuda'); g.manual_seed(1)
L = torch.empty((n, n), dtype=torch.float64, device='cuda'); L.uniform_(-1/n**0.5, 1/n**0.5, generator=g)
L.diagonal().uniform_(1.0, 2.0, generator=g)
V = torch.rand((k, n), dtype=torch.float64, device='cuda', generator=g) / n**0.5
for i in range(2):
    gcm.modify(L, V.clone(), 1 if i % 2 == 0 else -1, algo='panel')
torch.cuda.synchronize()
print('ok')
PY
python /tmp/pu.py > $out/plain.log 2>&1; }
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 2000 --csv --log-file $out/launches.csv python /tmp/pu.py > $out/ncu.log 2>&1
python tools/launches.py $out/launches.csv
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r02ad/launches.csv')))
st=next(i for i,r in enumerate(rows) if r and r[0]=="ID")
h=rows[st]; dur={}; grid={}
for r in rows[st+1:]:
    if len(r)!=len(h): continue
    d=dict(zip(h,r)); key=(d["ID"], d["Kernel Name"][:30])
    if d["Metric Name"]=="gpu__time_duration.sum": dur[key]=float(d["Metric Value"].replace(',',''))
    else: grid[key]=d["Metric Value"]
pu=[(grid[k],dur[k]) for k in dur if 'pupdate' in k[1]]
small=[t for g,t in pu if int(g.replace(',',''))<=8]
print("pupdate launches with <= 8 CTAs (lookahead):", len(small), "mean us", sum(small)/max(1,len(small)))
PY
