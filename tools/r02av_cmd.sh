out=gpurun_out/r02av; mkdir -p $out
cat > /tmp/bb.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_1011_1173_b200 as gcm
import synth, numpy as np
Ls, Vs, _ = synth.batched_instances(32, 512, 8, +1, first=0)
L = torch.from_numpy(np.tile(Ls, (128, 1, 1))).cuda(); V = torch.from_numpy(np.tile(Vs, (128, 1, 1))).cuda()
for i in range(3):
    gcm.modify_batched(L, V.clone(), 1 if i % 2 == 0 else -1)
torch.cuda.synchronize(); print('ok')
PY
python /tmp/bb.py > $out/plain.log 2>&1 && timeout 900 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --section Occupancy --import-source on --clock-control none -k regex:batched_tma -s 1 -c 1 -o $out/bt -f python /tmp/bb.py > $out/ncu.log 2>&1
echo rc=$?
