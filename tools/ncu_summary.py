"""Summarise an `ncu --set full` report into profiles/<tag>_ncu_summary.json.

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT.json "note"
Per kernel (first launch of each family): duration, DRAM bytes read/write (per launch),
SM / memory throughput, FP64 pipe utilisation, shared-memory wavefronts, grid, registers."""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "shared_wavefronts",
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "registers",
}
SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def family(name):
    for f in ("trsv", "btma", "btile", "bapply", "bdiag", "batched", "diag_chain", "panel_apply", "papply", "pupdate",
              "dsolve", "pinv", "pdiag", "ptile"):
        if f in name:
            return "bapply" if f in ("btma", "btile") else f
    return None


def from_long_csv(path):
    """An `ncu --csv --log-file` capture (one row per metric, e.g. application replay) as the
    wide (header, units, rows) form of `--page raw --csv`."""
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, mi, ui, vi, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"),
                          h.index("Metric Value"), h.index("ID"))
    per, units = {}, {}
    for r in rows[1:]:
        d = per.setdefault(r[ii], {"Kernel Name": r[ki]})
        d[r[mi]] = r[vi]
        units[r[mi]] = r[ui]
    hdr = ["Kernel Name"] + sorted(units)
    return hdr, [""] + [units[m] for m in hdr[1:]], [[d.get(c, "") for c in hdr] for d in per.values()]


def main(rep, out, note):
    if rep.endswith(".csv"):
        hdr, units, body = from_long_csv(rep)
        rows = [hdr, units] + body
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        fam = family(d.get("Kernel Name", ""))
        if fam is None or fam in res:
            continue
        k = {"kernel": d["Kernel Name"][:120]}
        for m, key in METRICS.items():
            if m not in d:
                continue
            v = d[m].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                continue
            u = units[hdr.index(m)]
            if key == "duration_us":
                x *= SCALE.get(u, 1.0)
            elif key.startswith("dram_bytes"):
                x *= SCALE.get(u, 1.0)
            k[key] = x
        if "dram_bytes_read" in k and "dram_bytes_write" in k:
            k["traffic_bytes"] = k["dram_bytes_read"] + k["dram_bytes_write"]
        res[fam] = k
    if "trsv" in res and "bapply" in res:  # bench.py's 'blocked' scope = TRSV kernel + overlapped Apply grid
        res["blocked"] = {"kernel": "trsv_kernel + btma_kernel (one profiling scope)",
                          "traffic_bytes": res["trsv"].get("traffic_bytes", 0) + res["bapply"].get("traffic_bytes", 0),
                          "duration_us_serialised": res["trsv"].get("duration_us", 0) + res["bapply"].get("duration_us", 0)}
    json.dump({"note": note, "kernels": res}, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
