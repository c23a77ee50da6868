out=gpurun_out/r02ac; mkdir -p $out
cat > /tmp/pu.py <<'PY'
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
python /tmp/pu.py > $out/plain.log 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:pupdate -s 60 -c 1 -o $out/pupdate -f python /tmp/pu.py > $out/ncu.log 2>&1
echo rc=$?
