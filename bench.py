#!/usr/bin/env python
"""Benchmark of the rank-k Cholesky up/down-date (arXiv 1011.1173) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME]

Prints ONE JSON line (rank 0).  A "step" is one pass of the whole hot path:
one in-place rank-k modification of the factor (SURVEY.md section 8(a) rows a0-a4,
through gcm_modify_ex), alternating update (sigma=+1) and downdate (sigma=-1) by
the same V so the factor stays bounded; V is restored from a pristine copy and
L2 is flushed (256 MiB write) between steps, outside the timed events.

Configs (BASELINE.json): "n5000_k16" (default, configs[1]: the metric's config),
"n5000_k1" / "n5000_k4" / "n5000_k64" (configs[2] sweep), "n100000_k32" (configs[3] at one
GPU: 80 GB factor drawn on the device, column-norm pin at full size), "batched" (configs[4]:
4096 factors n=512, k=8; weak-sharded over ranks).

--impl reference times the CPU oracle (oracle/, plain serial C) on the same
workload as the reference arm (rank 0 only).
"""
from __future__ import annotations

import argparse
import contextlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")  # no version banner: the JSON line is the only stdout line

import numpy as np  # noqa: E402

METRIC = "rank-k modify ms & fp64 GFLOP/s (n=5000,k=16); % of HBM/FP64 roofline"
# FP64 vector peak derived from the unit counts and clock (B200_PROFILING.md: 148 SMs,
# 1965 MHz max; 64 FP64 FMA/clk/SM): 148*64*2*1.965e9 -- the fallback when no measured
# figure is committed.  The measured one is tools/fp64_peak.cu's JSON line, committed as
# profiles/*fp64_peak*.json.
FP64_PEAK_TFLOPS_DERIVED = 148 * 64 * 2 * 1.965e9 / 1e12

CONFIGS = {
    "n5000_k16": dict(n=5000, k=16),
    "n5000_k1": dict(n=5000, k=1),
    "n5000_k4": dict(n=5000, k=4),
    "n5000_k64": dict(n=5000, k=64),
    "batched": dict(n=512, k=8, batch=4096),
    # BASELINE configs[3] at one GPU: 80 GB factor, direct-L construction generated on the
    # device (R18), checked by the column-norm identity at full size
    "n100000_k32": dict(n=100000, k=32, direct=True),
    # BASELINE configs[3] column-sharded over the job's GPUs (gcm_modify_dist, NCCL; nb = 512
    # block-cyclic columns); strong scaling: the same 80 GB factor for every N
    "n100000_k32_dist": dict(n=100000, k=32, direct=True, dist=True, nb=512),
}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def fp64_peak():
    """(TFLOP/s, source, link latencies) from the newest committed tools/fp64_peak.cu output."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_fp64_peak.json")))
    if files:
        try:
            d = json.load(open(files[-1]))
            return float(d["fp64_tflops"]), f"measured ({os.path.basename(files[-1])}, tools/fp64_peak.cu)", d
        except Exception:
            pass
    return FP64_PEAK_TFLOPS_DERIVED, "derived (148 SM x 64 FMA/clk x 2 x 1.965 GHz)", {}


def chain_floor(n, k, links, sm_mhz):
    """SURVEY 8(d) latency bound beside the roofline: T_chain = (n + k - 1) t_link for the
    literal sweep (the paper's Compute link, sqrt + div, measured by tools/fp64_peak.cu), and
    this path's own serial chain: ceil(n/32) TRSV steps, each at least one inter-SM hand-off
    (one-way relaxed store -> polling load, tools/pingpong.cu: 750 cycles)."""
    mhz = sm_mhz or 1965.0
    t_link = links.get("t_link_compute_cycles")
    out = {"clock_mhz": mhz}
    if t_link:
        out["literal_sweep"] = {"links": n + k - 1, "t_link_cycles": t_link,
                                "ms": round((n + k - 1) * t_link / mhz / 1e3, 4)}
    steps = (n + 31) // 32
    out["blocked_trsv"] = {"steps": steps, "t_step_floor_cycles": 750,
                           "ms": round(steps * 750 / mhz / 1e3, 4),
                           "note": "one inter-SM hand-off per 32-row TRSV step (tools/pingpong.cu)"}
    return out


def algorithmic(n, k, batch=1):
    """Algorithmic units of one step: Apply count, flops, HBM bytes."""
    applies = batch * k * n * (n - 1) // 2
    flops = 6 * applies
    bytes_ = batch * (8 * n * (n + 1) + 16 * n * k)  # upper triangle read+write, V read+write
    return applies, flops, bytes_


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled every 1 ms through NVML (the
    library nvidia-smi reads) on a thread that runs DURING the timed region; the
    region is only entered once the first sample has arrived.  Falls back to
    `nvidia-smi -lms 200` when NVML is unavailable."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, device_index):
        self.device_index = device_index
        self.rows = []
        self.stop_evt = threading.Event()
        self.thread = None
        self.handle = None
        self.nvml = None
        self.smax = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            handle = None
            try:
                import torch
                pr = torch.cuda.get_device_properties(self.device_index)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                handle = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                handle = pynvml.nvmlDeviceGetHandleByIndex(self.device_index)
            self.nvml, self.handle = pynvml, handle
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(handle, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
            t0 = time.perf_counter()
            while not self.rows and time.perf_counter() - t0 < 2.0:
                time.sleep(0.001)
        except Exception:
            self.nvml = None

    def _run(self):
        nv, h = self.nvml, self.handle
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop_evt.is_set():
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), int(get_reasons(h))))
            except Exception:
                pass
            time.sleep(0.001)

    def mark(self):
        """Index of the first sample taken after this call (start of the timed region)."""
        return len(self.rows)

    def stop(self, first=0):
        if self.nvml is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self.stop_evt.set()
        self.thread.join(timeout=1)
        rows = self.rows[first:] or self.rows[-1:]
        sm = [r[0] for r in rows]
        reasons = sorted({name for _, bits in rows for bit, name in self.REASONS.items() if bits & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax, "reasons": reasons,
                "samples": len(rows), "source": "nvml, 1 ms period, timed region only"}


def dist_setup(ngpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        import torch
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- our arm
def run_ours(args, world, rank, local):
    import torch
    import paper_1011_1173_b200 as gcm
    import synth

    cfg = CONFIGS[args.config]
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    n, k = cfg["n"], cfg["k"]
    batch = cfg.get("batch", 1)
    stream = torch.cuda.current_stream(dev)

    comm = gcols = None
    if cfg.get("dist"):
        # this rank's block-cyclic shard of the direct-L instance (R18), drawn on the
        # device: row c of L is global column gcols[c] (its entries above the diagonal
        # (2U-1)/sqrt(n), diagonal U[1,2)), V rows U/sqrt(n)
        from paper_1011_1173_b200 import dist as gdist
        nb = cfg["nb"]
        gcols_np = gdist.global_cols(n, nb, world, rank)
        gcols = torch.from_numpy(gcols_np).to(dev)
        g = torch.Generator(device=dev)
        g.manual_seed(synth.SEED_ROOT + 1000 + rank)
        L = torch.empty((len(gcols_np), n), dtype=torch.float64, device=dev)
        L.uniform_(-1.0 / n ** 0.5, 1.0 / n ** 0.5, generator=g)
        rows = torch.arange(len(gcols_np), device=dev)
        L[rows, gcols] = 1.0 + torch.rand(len(gcols_np), dtype=torch.float64, device=dev, generator=g)
        V0 = torch.rand((k, len(gcols_np)), dtype=torch.float64, device=dev, generator=g) / n ** 0.5
        Lbuf = Vbuf = None
        comm = gdist.Comm(rank, world)
    elif cfg.get("direct"):
        # direct-L instance (R18) drawn on the device with torch's seeded Philox
        # generator: L_ii ~ U[1,2), L_ij ~ (2U-1)/sqrt(n), V ~ U/sqrt(n); update then downdate
        g = torch.Generator(device=dev)
        g.manual_seed(synth.SEED_ROOT + rank)
        L = torch.empty((n, n), dtype=torch.float64, device=dev)
        L.uniform_(-1.0 / n ** 0.5, 1.0 / n ** 0.5, generator=g)
        L.diagonal().uniform_(1.0, 2.0, generator=g)
        V0 = torch.rand((k, n), dtype=torch.float64, device=dev, generator=g) / n ** 0.5
        Lbuf = Vbuf = None
    elif batch == 1:
        Lbuf, Vbuf, _ = synth.paper_instance(n, k, +1, seed=synth.SEED_ROOT + rank)
        L = torch.from_numpy(Lbuf).to(dev)
        V0 = torch.from_numpy(Vbuf).to(dev)
    else:
        per = batch // world  # weak sharding: each rank owns its slice of the factors
        distinct = min(per, 32)  # distinct seeded factors, tiled to fill the slice
        Ls, Vs, _ = synth.batched_instances(distinct, n, k, +1, first=rank * per)
        reps = (per + distinct - 1) // distinct
        L = torch.from_numpy(np.tile(Ls, (reps, 1, 1))[:per].copy()).to(dev)
        V0 = torch.from_numpy(np.tile(Vs, (reps, 1, 1))[:per].copy()).to(dev)
        batch = per
    V = V0.clone()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def call(sigma):
        if comm is not None:
            gdist.modify_dist(comm, L, V, n, cfg["nb"], sigma)
        elif batch == 1:
            gcm.modify(L, V, sigma, algo=args.algo)
        else:
            gcm.modify_batched(L, V, sigma)

    # warm-up
    for i in range(args.warmup):
        V.copy_(V0)
        call(+1 if i % 2 == 0 else -1)
    torch.cuda.synchronize()
    gcm.profile_read()
    gcm.profile_launches()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    gcm.profile_enable(True)
    barrier(world)
    torch.cuda.synchronize()
    first_sample = clocks.mark()
    t0 = time.perf_counter()
    for i in range(args.steps):
        V.copy_(V0)
        flush.fill_(float(i))  # L2 flush: 256 MiB write, outside the step's events
        ev[i][0].record(stream)
        call(+1 if i % 2 == 0 else -1)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    barrier(world)
    wall = time.perf_counter() - t0
    gcm.profile_enable(False)
    prof = gcm.profile_read()
    clk = clocks.stop(first_sample)
    check = None
    if cfg.get("direct"):
        # full-size property pin: ||L~_{:,c}||^2 = ||L_{:,c}||^2 + sigma ||V_{c,:}||^2
        # on 256 sampled (local) columns, one more (untimed) update
        nl = L.shape[0]
        cols = torch.randperm(nl, device=dev, generator=torch.Generator(device=dev).manual_seed(7))[:256]
        gc = gcols[cols] if gcols is not None else cols
        mask = torch.arange(n, device=dev)[None, :] <= gc[:, None]
        before = ((L[cols] * mask) ** 2).sum(1)
        V.copy_(V0)
        vnorm = (V0[:, cols] ** 2).sum(0)
        call(+1)
        torch.cuda.synchronize()
        after = ((L[cols] * mask) ** 2).sum(1)
        rel = ((after - before - vnorm).abs() / after).max().item()
        check = {"pin": "column-norm identity on 256 sampled columns (SURVEY 8(c) P4)",
                 "max_rel_err": rel, "ok": rel <= 1e-11}

    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = max_over_ranks(sum(step_ms), world)
    ms_per_step = total_ms / args.steps
    applies, flops, bytes_ = algorithmic(n, k, batch)
    # GFLOP/s of the whole job: replicas / factor shards (weak) add up; one sharded factor (strong) does not
    value = (1 if comm is not None else world) * flops / (ms_per_step * 1e-3) / 1e9

    # dominant kernel and its roofline (bytes/flops per launch from DESIGN.md "roofline")
    hbm, hbm_src = measured_peaks()
    # kernels per profiling scope: 'blocked' = trsv_kernel + its programmatic-dependent btma_kernel
    launches = gcm.profile_launches()  # counted by the library at every launch site
    dom = max(prof.items(), key=lambda kv: kv[1][1]) if prof else ("none", (1, 0.0))
    dname, (dcount, dms) = dom
    per_launch_ms = dms / max(dcount, 1)
    # launches of the dominant scope per step: k > 32 runs ceil(k/32) passes (R3),
    # each launch does 1/passes of the step's work
    per_step = max(1, round(dcount / args.steps))
    kb = kernel_units(dname, n, k, batch, per_step)
    f64, f64_src, links = fp64_peak()
    if kb["bound"] == "hbm":
        achieved = kb["bytes"] / (per_launch_ms * 1e-3) / 1e9
        peak, unit = hbm, "GB/s"
    else:
        achieved = kb["flops"] / (per_launch_ms * 1e-3) / 1e12
        peak, unit = f64, "TFLOP/s"
    traffic = ncu_traffic(dname, args.config)
    roofline = {"kernel": dname, "bound": kb["bound"], "achieved": round(achieved, 3), "peak": peak,
                "peak_source": hbm_src if kb["bound"] == "hbm" else f64_src,
                "unit": unit, "frac": round(achieved / peak, 4),
                "traffic": traffic["bytes"] if traffic else None,
                "traffic_source": traffic["source"] if traffic else None,
                "algorithmic_bytes": kb["bytes"], "algorithmic_flops": kb["flops"], "launches_per_step": per_step,
                "algorithmic": kb["what"], "share_of_step": round(dms / max(sum(m for _, m in prof.values()), 1e-9), 3)}
    # whole-path roofline: T_roof = max(flops/F64, bytes/HBM)
    t_roof = max(flops / (f64 * 1e12), bytes_ / (hbm * 1e9))
    roofline_path = {"t_roof_ms": round(t_roof * 1e3, 4), "t_step_ms": round(ms_per_step, 4),
                     "frac": round(t_roof * 1e3 / ms_per_step, 4),
                     "bound": "fp64" if flops / f64 / 1e12 > bytes_ / hbm / 1e9 else "hbm",
                     "achieved_gbs": round(bytes_ / (ms_per_step * 1e-3) / 1e9, 1),
                     "achieved_gflops": round(flops / (ms_per_step * 1e-3) / 1e9, 1)}

    out = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "strong" if comm is not None else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config, n, k, batch * world),
                   "n": n, "k": k, "batch_per_gpu": batch,
                   "algo": "dist (gcm_modify_dist, NCCL)" if comm is not None else (args.algo if batch == 1 else "batched"),
                   "sigma": "alternating +1/-1 by the same V", "l2": "flushed between steps (256 MiB write)",
                   "parallelism": (f"column-sharded x{world} (block-cyclic nb={cfg['nb']})" if comm is not None else
                                   f"replicas x{world}" if batch == 1 else f"factor-sharded x{world}"),
                   "instance": ("direct-L (DESIGN.md R18) on the device, torch Philox seed 10111173+rank"
                                if cfg.get("direct") else
                                "paper construction (PAPER.md 111): B,V ~ U[0,1), A = B^T B + I, seed 10111173+rank")},
        "roofline": roofline, "roofline_path": roofline_path,
        "chain_floor": chain_floor(n, k, links, clk.get("sm_mhz")) if batch == 1 else None,
        "gpu_launches": int(launches),
        "kernels": {kname: {"launches": c, "ms_total": round(m, 4)} for kname, (c, m) in prof.items()},
        "clocks": clk, "wall_s": round(wall, 4),
    }
    if check is not None:
        out["check"] = check
    if rank == 0 and batch == 1 and not args.no_e2e and Lbuf is not None:
        out["e2e"] = run_e2e(gcm, torch, Lbuf, Vbuf, n, k, flops)
    if batch > 1 and not args.no_e2e:  # every rank its own slice, max over ranks
        e2e = run_e2e_batched(gcm, torch, L, V0, flops, world)
        if rank == 0:
            out["e2e"] = e2e
    if rank == 0 and not args.no_cpu:
        out["cpu_baseline"] = run_cpu_baseline(n, k)
    return out


def ncu_traffic(kernel, config):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`, from the newest
    committed `ncu --set full` summary OF THIS CONFIG (profiles/r*_ncu_<config>.json, written
    by tools/ncu_summary.py from a capture of `bench.py --config <config>`), else None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_ncu_{config}.json")))
    if not files and config == "n5000_k16":
        files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_summary.json")))
    if not files:
        return None
    try:
        d = json.load(open(files[-1]))["kernels"].get(kernel)
        if d is None or d.get("traffic_bytes") is None:
            return None
        return {"bytes": d["traffic_bytes"], "source": os.path.basename(files[-1])}
    except Exception:
        return None


def kernel_units(name, n, k, batch, per_step=1):
    """Algorithmic work of ONE launch of each kernel family.  A step
    with k > 32 runs ceil(k/32) passes (per_step launches of the same scope): each launch
    carries its pass's share of the update columns (the triangle is read and written once
    PER PASS, so the bytes are per pass too)."""
    tri = 8 * n * (n + 1) // 2  # bytes of the upper triangle
    kp = k / per_step  # update columns per launch (average)
    if name in ("blocked", "pchain"):  # solve chain + sweeps + the Apply overlapped with it (one scope)
        return {"bound": "hbm" if kp < 16 else "alu", "bytes": 8 * n * (n + 1) + 16 * n * kp,
                "flops": 6 * kp * n * (n - 1) / 2,
                "what": f"one pass of {kp:g} update columns (TRSV + fused sweeps + overlapped Apply): upper "
                        "triangle read+write once + V; 6 flops per Apply"}
    if name == "ptrsv":  # panel algorithm's right-looking solve: the triangle read once, k FMA per element
        return {"bound": "alu" if kp >= 16 else "hbm", "bytes": tri + 16 * n * kp, "flops": n * n * kp,
                "what": "column-block solve + residual updates: L triangle read once, n^2 k flops (2 per FMA)"}
    if name == "papply":  # panel algorithm's Apply: every tile read+written once, 6 flops per Apply
        return {"bound": "hbm" if kp < 16 else "alu", "bytes": 2 * tri, "flops": 6 * kp * n * (n - 1) / 2,
                "what": "upper triangle read+write once (off-diagonal tiles); 6 flops per Apply"}
    if name == "trsv":  # reads the triangle once for P = L^-T V (k FMA per element)
        return {"bound": "hbm", "bytes": tri + 16 * n * kp, "flops": n * n * kp,
                "what": "L triangle read once + V read + P write; n^2 k flops"}
    if name == "bapply":  # off-diagonal tiles read+write once, 2k FMA per element
        off = 2 * tri * (1 - 64.0 / n)
        return {"bound": "hbm" if kp < 16 else "alu", "bytes": off, "flops": 6 * kp * n * (n - 1) / 2 * (1 - 64.0 / n),
                "what": "off-diagonal triangle read+write; 6 flops per Apply"}
    if name == "panel_apply":
        return {"bound": "hbm", "bytes": 2 * tri / max(1, (n + 63) // 64), "flops": 6 * kp * n * 64 / 2,
                "what": "one 64-row panel read+write (average)"}
    if name == "batched":
        return {"bound": "hbm", "bytes": batch * (2 * tri + 16 * n * k), "flops": batch * 6 * k * n * (n - 1) / 2,
                "what": "every factor's triangle read+write once, V read+write"}
    return {"bound": "hbm", "bytes": 0, "flops": 0, "what": "unmodelled"}


def workload_name(cfg, n, k, total_batch):
    if total_batch > 1:
        return f"batched {total_batch} x (n={n}, k={k}) fp64 update/downdate"
    return f"n={n}, k={k} fp64 rank-k update/downdate (BASELINE configs[1])" if (n, k) == (5000, 16) else \
        f"n={n}, k={k} fp64 rank-k update/downdate"


def run_e2e(gcm, torch, Lbuf, Vbuf, n, k, flops, steps=3):
    """Same metric through the C-ABI with HOST buffers (gcm_modify_host): H2D + modify + D2H per step."""
    Lh = torch.from_numpy(Lbuf.copy()).pin_memory()
    Vh0 = torch.from_numpy(Vbuf.copy())
    Vh = Vh0.clone().pin_memory()
    ts = []
    for i in range(steps + 1):
        Vh.copy_(Vh0)
        t0 = time.perf_counter()
        gcm.modify_host(Lh, Vh, +1 if i % 2 == 0 else -1)
        dt = time.perf_counter() - t0
        if i > 0:
            ts.append(dt)
    t = statistics.median(ts)
    nb = gcm.modify_host_bytes(n, k)  # upper-triangle column blocks + V, each direction
    return {"value": round(flops / t / 1e9, 2), "unit": "GFLOP/s", "ms_per_step": round(t * 1e3, 3),
            "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb, "api": "gcm_modify_host (pinned host L, V)"}


def run_e2e_batched(gcm, torch, L, V0, flops, world, steps=3):
    """Batched e2e through gcm_modify_batched: each step copies every factor's L and V from
    pinned host memory to the device, modifies, and copies both back (whole matrices: the
    batched API takes full n x n buffers)."""
    Lh = L.cpu().pin_memory()
    Vh0 = V0.cpu()
    Vh = Vh0.clone().pin_memory()
    Ld = torch.empty_like(L)
    Vd = torch.empty_like(V0)
    ts = []
    for i in range(steps + 1):
        Vh.copy_(Vh0)
        torch.cuda.synchronize()
        barrier(world)
        t0 = time.perf_counter()
        Ld.copy_(Lh, non_blocking=True)
        Vd.copy_(Vh, non_blocking=True)
        gcm.modify_batched(Ld, Vd, +1 if i % 2 == 0 else -1)
        Lh.copy_(Ld, non_blocking=True)
        Vh.copy_(Vd, non_blocking=True)
        torch.cuda.synchronize()
        dt = max_over_ranks(time.perf_counter() - t0, world)
        if i > 0:
            ts.append(dt)
    t = statistics.median(ts)
    nbytes = (L.numel() + V0.numel()) * 8 * world
    return {"value": round(flops * world / t / 1e9, 2), "unit": "GFLOP/s", "ms_per_step": round(t * 1e3, 3),
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
            "api": "gcm_modify_batched with pinned-host L, V copied in and out every step"}


def run_cpu_baseline(n, k, budget_s=20.0):
    """The oracle (plain serial C, oracle/) on this host: bounded sample of the same workload."""
    import oracle
    import synth
    cores = 1  # the oracle is single-threaded by construction
    sample_note = ""
    if n > 20000:  # bounded sample: the same construction at n = 4000 (the oracle is O(n^2 k) serial)
        n = 4000
        Lbuf, Vbuf = synth.direct_instance(n, k, seed=synth.SEED_ROOT)
        sample_note = " (direct-L construction, leading-size sample of the n=100000 workload)"
    else:
        Lbuf, Vbuf, _ = synth.paper_instance(n, k, +1, seed=synth.SEED_ROOT)
    calls, t_tot = 0, 0.0
    while t_tot < budget_s and calls < 4:
        L = Lbuf.copy()
        V = Vbuf.copy()
        t0 = time.perf_counter()
        oracle.modify_a(L, V, +1)
        t_tot += time.perf_counter() - t0
        calls += 1
        if t_tot > budget_s / 4:
            break
    _, flops, _ = algorithmic(n, k)
    return {"value": round(flops * calls / t_tot / 1e9, 3), "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
            "sample": f"{calls} full oracle call(s) of n={n}, k={k} update ({t_tot:.2f} s){sample_note}",
            "ms_per_call": round(t_tot / calls * 1e3, 1)}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, world, rank):
    """Reference arm: the CPU oracle, as it stands, on the host cores (rank 0 only)."""
    import oracle
    import synth
    cfg = CONFIGS[args.config]
    n, k = cfg["n"], cfg["k"]
    batch = cfg.get("batch", 1)
    if batch > 1:
        n_use, k_use, calls_per_step = n, k, 16  # bounded sample: 16 factors per step
    else:
        n_use, k_use, calls_per_step = n, k, 1
    Lbuf, Vbuf, _ = synth.paper_instance(n_use, k_use, +1, seed=synth.SEED_ROOT)
    L = Lbuf.copy()

    def step(i):
        for _ in range(calls_per_step):
            V = Vbuf.copy()
            oracle.modify_a(L, V, +1 if i % 2 == 0 else -1)

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(i)
    t = time.perf_counter() - t0
    _, flops, _ = algorithmic(n_use, k_use, calls_per_step)
    value = flops * args.steps / t / 1e9
    sample = (f"{calls_per_step} oracle call(s) of n={n_use}, k={k_use} per step"
              + (f" (bounded sample of the {batch}-factor batch)" if batch > 1 else ""))
    return {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.config, n, k, batch), "n": n, "k": k},
            "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


@contextlib.contextmanager
def stdout_to_stderr():
    """File descriptor 1 -> 2 while the run executes: whatever native libraries print (NCCL's
    version banner ignores NCCL_DEBUG on some boxes) goes to stderr, so the JSON line is the
    only line bench.py writes to stdout."""
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        yield
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="n5000_k16")
    ap.add_argument("--algo", choices=["auto", "sweep", "blocked", "panel"], default="auto")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, world, rank)), flush=True)
        return
    with stdout_to_stderr():  # library banners (NCCL's version line) must not precede the JSON line
        world, rank, local = dist_setup(args.gpus)
        out = run_ours(args, world, rank, local)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        with stdout_to_stderr():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
