"""Summarise ncu captures into profiles/ (committed evidence).

python tools/ncu_summary.py <full.ncu-rep> <launches.csv> <out_prefix> [n]

Writes <out_prefix>_ncu_summary.md (per-kernel metrics of the full capture
and each kernel's share of the step from the launch list) and updates
profiles/ncu_traffic.json (DRAM bytes per launch per pipeline stage, read by
bench.py for the roofline "traffic" field).
"""

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

STAGE_OF = [("k_descent", "local"), ("k_mr2d", "local"), ("k_lce", "local"),
            ("k_update_local", "fused"), ("k_row_fwd", "row_fwd"), ("k_row_inv", "row_inv"),
            ("k_grad", "grad"), ("k_res_march", "grad"), ("k_colp<", None), ("k_col<", None)]
METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "lts__t_bytes.sum": "l2_bytes",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
        "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0}


def stage_of(name, col_idx):
    for key, st in STAGE_OF:
        if key in name:
            if st is None:
                # k_col<N1, N2, MODE>: MODE 0 fwd, 1 inv, 2 solve
                key_ = "k_colp<" if "k_colp<" in name else "k_col<"
                mode = name.split(key_, 1)[1].split(">")[0].split(",")[-1].strip()
                return {"0": "col_fwd", "1": "col_inv", "2": "col_solve"}.get(mode, "col")
            return st
    return "other"


def load_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"name": r[hdr.index("Kernel Name")]}
        for m, k in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[k] = v * UNIT.get(units[i], 1.0)
        res.append(d)
    return res


def load_launches(path):
    per = defaultdict(float)
    cnt = defaultdict(int)
    other = defaultdict(float)
    with open(path) as f:
        txt = f.read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        st = stage_of(r[ki], 0)
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        per[st] += v
        cnt[st] += 1
        if st == "other":
            other[r[ki].split("(")[0].split("<")[0].replace("void ", "").strip()] += v
    load_launches.other = other
    return per, cnt


def main():
    rep, launches, prefix = sys.argv[1:4]
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 256
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    sb = bench.stage_bytes(n)
    kernels = load_raw(rep)
    lines = [f"# ncu summary ({os.path.basename(prefix)}), grid {n}^3, config-2 laminate", "",
             "Full capture (`--set full --clock-control none`), one launch per stage kernel:", "",
             "| kernel | stage | us | DRAM read MB | DRAM write MB | traffic / alg. bytes | DRAM % | "
             "SM % | occupancy % | FP64 pipe % | regs |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for k in kernels:
        st = stage_of(k["name"], 0)
        tr = k.get("dram_read", 0) + k.get("dram_write", 0)
        alg = sb.get(st)
        traffic[st] = tr
        lines.append(
            f"| `{k['name'][:60]}` | {st} | {k.get('duration', 0) * 1e6:.1f} | "
            f"{k.get('dram_read', 0) / 1e6:.1f} | {k.get('dram_write', 0) / 1e6:.1f} | "
            f"{(tr / alg) if alg else float('nan'):.3f} | {k.get('dram_pct', 0):.1f} | "
            f"{k.get('sm_pct', 0):.1f} | {k.get('occupancy_pct', 0):.1f} | "
            f"{k.get('fp64_pipe_pct', 0):.1f} | {int(k.get('regs', 0))} |")
    if launches and os.path.exists(launches):
        per, cnt = load_launches(launches)
        tot = sum(per.values())
        lines += ["", "Launch list (`--metrics gpu__time_duration.sum`, cold-cache, serialised): "
                  "share of kernel time per stage", "", "| stage | launches | total us | share |",
                  "|---|---|---|---|"]
        for st, v in sorted(per.items(), key=lambda x: -x[1]):
            lines.append(f"| {st} | {cnt[st]} | {v * 1e6:.1f} | {v / tot:.3f} |")
        oth = getattr(load_launches, "other", {})
        if oth:
            lines += ["", "`other` = kernels outside the iteration (host-transfer AoS/SoA transposes of "
                      "setup and of the e2e leg, det checks, field sums):", "",
                      "| kernel | total us |", "|---|---|"]
            for k, v in sorted(oth.items(), key=lambda x: -x[1])[:8]:
                lines.append(f"| `{k}` | {v * 1e6:.1f} |")
    with open(prefix + "_ncu_summary.md", "w") as f:
        f.write("\n".join(lines) + "\n")
    tpath = os.path.join(os.path.dirname(prefix), "ncu_traffic.json")
    with open(tpath, "w") as f:
        json.dump({k: v for k, v in traffic.items()}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
