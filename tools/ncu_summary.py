"""Summarise a bench capture for profiles/: one row per stage kernel from a
`ncu --set full` report (DRAM bytes vs the stage's algorithmic bytes, DRAM /
SM / FP64-pipe utilisation, occupancy, registers), the per-stage share of a
`--metrics gpu__time_duration.sum` launch list, and the per-launch DRAM
traffic map bench.py reads (profiles/ncu_traffic.json).

usage: python tools/ncu_summary.py FULL.ncu-rep LAUNCHES.csv OUT.md [n]
"""
import csv
import io
import json
import subprocess
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

STAGE_OF = [("k_update_local", "fused"), ("k_row_fwd", "row_fwd"), ("k_row_inv", "row_inv"),
            ("k_plane", "plane"), ("k_res_march", "grad"), ("k_grad", "grad"),
            ("k_descent", "local"), ("k_colp<16, 16, 0>", "col_fwd"),
            ("k_colp<16, 16, 1>", "col_inv"), ("k_col<", "col_solve")]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-3, "us": 1.0, "ms": 1e3,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}


def stage(name):
    for key, st in STAGE_OF:
        if key in name:
            return st
    return "other"


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            try:
                d[h] = float(v.replace(",", "")) * SCALE.get(u, 1.0)
            except ValueError:
                d[h] = v
        res.append(d)
    return res


def main():
    rep, launches, out_md = sys.argv[1:4]
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 256
    alg = bench.stage_bytes(n)
    rows = raw_rows(rep)
    lines = [f"# ncu summary, grid {n}^3, config-2 laminate (bench.py --steps 8 --warmup 3; launch list --steps 3)", "",
             "Full capture (`--set full --clock-control none`), one launch per stage kernel:", "",
             "| kernel | stage | us | DRAM read MB | DRAM write MB | traffic / alg. bytes | DRAM % "
             "| SM % | warps active % | FP64 pipe % | regs |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for d in rows:
        name = d["Kernel Name"]
        st = stage(name)
        rd, wr = d["dram__bytes_read.sum"], d["dram__bytes_write.sum"]
        ratio = (rd + wr) / alg[st] if st in alg else float("nan")
        traffic.setdefault(st, rd + wr)
        lines.append(
            f"| `{name[:60]}` | {st} | {d['gpu__time_duration.sum']:.1f} | {rd / 1e6:.1f} | "
            f"{wr / 1e6:.1f} | {ratio:.3f} | "
            f"{d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']:.1f} | "
            f"{d['sm__throughput.avg.pct_of_peak_sustained_elapsed']:.1f} | "
            f"{d['sm__warps_active.avg.pct_of_peak_sustained_active']:.1f} | "
            f"{d['sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active']:.1f} | "
            f"{int(d['launch__registers_per_thread'])} |")
    # launch list: share of kernel time per stage
    tot, per, cnt = 0.0, {}, {}
    with open(launches) as f:
        txt = f.read()
    rr = list(csv.reader(io.StringIO(txt[txt.index('"ID"'):])))
    h = rr[0]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    for r in rr[1:]:
        if len(r) <= iv:
            continue
        us = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
        st = stage(r[ik])
        per[st] = per.get(st, 0.0) + us
        cnt[st] = cnt.get(st, 0) + 1
        tot += us
    lines += ["", "Launch list (`--metrics gpu__time_duration.sum`, serialised): share of kernel "
              "time per stage", "", "| stage | launches | total us | share |", "|---|---|---|---|"]
    for st, us in sorted(per.items(), key=lambda kv: -kv[1]):
        lines.append(f"| {st} | {cnt[st]} | {us:.1f} | {us / tot:.3f} |")
    open(out_md, "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
