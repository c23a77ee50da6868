out=gpurun_out/r02ao; mkdir -p $out
cat > /tmp/b5.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_1011_1173_b200 as gcm
import synth
Lb, Vb, _ = synth.paper_instance(5000, 16, 1)
L = torch.from_numpy(Lb).cuda(); V = torch.from_numpy(Vb).cuda()
for i in range(4):
    gcm.modify(L, V.clone(), 1, algo='blocked')
torch.cuda.synchronize(); print('ok')
PY
python /tmp/b5.py > $out/plain.log 2>&1 && timeout 600 ncu --section SourceCounters --section WarpStateStats --import-source on --clock-control none -k regex:trsv_kernel -s 2 -c 1 -o $out/trsv -f python /tmp/b5.py > $out/ncu.log 2>&1
echo rc=$?
