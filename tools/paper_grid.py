"""The paper's experimental grid (PAPER.md 111-115, Figs. 2 and 3) on B200: an n-sweep at
k in {16, 1}, single and double precision, update and downdate, reporting time and the
paper's error metric max_ij |A~_ij - (L~^T L~)_ij| (C computed with fp64 BLAS) beside the
relative Frobenius difference from the fp64 oracle, for the GPU path (gcm_modify for fp64,
gcm_modify_f32 for fp32) and the CPU oracle (serial C; fp64 / fp32) where it fits the time
budget.  Instances: the paper's construction (B, V ~ U[0,1), A = B^T B + I [+ V V^T]).

    python tools/paper_grid.py [--ns 500,1000,2000,3000,4000,5000] [--out profiles/r02_paper_grid]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1011_1173_b200 as gcm  # noqa: E402
import synth  # noqa: E402
from gcm_testutil import rel_fro, upper  # noqa: E402


def paper_error(At_dev, Lt):
    """max|A~ - L~^T L~| with the product in fp64 on the GPU (the paper: 'computed with the BLAS')."""
    U = torch.from_numpy(np.triu(Lt[:, :Lt.shape[0]].T).astype(np.float64)).cuda()
    return float((At_dev - U.T @ U).abs().max().item())


def gpu_time(fn, reps=3):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        prep = fn(None)
        a.record()
        fn(prep)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="500,1000,2000,3000,4000,5000")
    ap.add_argument("--cpu-max-n", type=int, default=2000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_paper_grid"))
    args = ap.parse_args()
    rows = []
    for k in (16, 1):
        for n in [int(x) for x in args.ns.split(",")]:
            for sigma in (1, -1):
                Lbuf, Vbuf, A = synth.paper_instance(n, k, sigma, seed=synth.SEED_ROOT + n + k)
                At = A + sigma * (Vbuf.T @ Vbuf)
                At_dev = torch.from_numpy(At).cuda()
                L64, V64 = Lbuf.copy(), Vbuf.copy()
                t0 = time.perf_counter()
                if n <= args.cpu_max_n:
                    oracle.modify_a(L64, V64, sigma)
                    cpu64 = time.perf_counter() - t0
                else:  # the fp64 reference result still comes from the oracle, untimed budget aside
                    oracle.modify_a(L64, V64, sigma)
                    cpu64 = None
                for prec in ("f64", "f32"):
                    dt = np.float64 if prec == "f64" else np.float32
                    Ld = torch.from_numpy(Lbuf.astype(dt)).cuda()
                    Vd = torch.from_numpy(Vbuf.astype(dt)).cuda()
                    out = {}

                    def fn(prep):
                        if prep is None:
                            return (Ld.clone(), Vd.clone())
                        L, V = prep
                        (gcm.modify if prec == "f64" else gcm.modify_f32)(L, V, sigma)
                        out["L"] = L
                    ms = gpu_time(fn)
                    Lg = out["L"].cpu().numpy()
                    row = {"k": k, "n": n, "op": "update" if sigma > 0 else "downdate", "prec": prec,
                           "gpu_ms": round(ms, 4), "gpu_err": paper_error(At_dev, Lg),
                           "gpu_relF_vs_f64_oracle": rel_fro(upper(Lg).astype(np.float64), upper(L64))}
                    if prec == "f64":
                        row["cpu_ms"] = None if cpu64 is None else round(cpu64 * 1e3, 1)
                        row["cpu_err"] = paper_error(At_dev, L64)
                    elif n <= args.cpu_max_n:
                        L32, V32 = Lbuf.astype(np.float32), Vbuf.astype(np.float32)
                        t0 = time.perf_counter()
                        oracle.modify_a_f32(L32, V32, sigma)
                        row["cpu_ms"] = round((time.perf_counter() - t0) * 1e3, 1)
                        row["cpu_err"] = paper_error(At_dev, L32)
                    rows.append(row)
                    print(json.dumps(row), flush=True)
    with open(args.out + ".jsonl", "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
    with open(args.out + ".md", "w") as f:
        f.write("# Paper grid (PAPER.md 111, Figs. 2-3) on B200: time and max|A~ - L~^T L~|\n\n")
        f.write("GPU = this library (fp64: gcm_modify, auto algorithm; fp32: gcm_modify_f32); CPU = the serial C "
                "oracle on one host core (the paper's CPU side was LAPACK/LINPACK; context only).\n\n")
        f.write("| k | n | op | prec | GPU ms | CPU ms | GPU err | CPU err | GPU rel-F vs fp64 oracle |\n")
        f.write("|---|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            f.write(f"| {r['k']} | {r['n']} | {r['op']} | {r['prec']} | {r['gpu_ms']} | {r.get('cpu_ms')} | "
                    f"{r['gpu_err']:.3e} | {r.get('cpu_err', float('nan')):.3e} | {r['gpu_relF_vs_f64_oracle']:.2e} |\n")


if __name__ == "__main__":
    main()
