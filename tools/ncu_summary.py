"""Summarise ncu captures into profiles/ (tracked): per-launch key metrics,
top stall reasons, and the launch-list share per kernel.

    python tools/ncu_summary.py --rep gpurun_out/prof_pull_r1.ncu-rep ... \
        --launches gpurun_out/launches_mega.csv --out profiles/r01_summary.md \
        --traffic profiles/traffic.json
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("lts__t_sector_hit_rate.pct", "L2_hit_%"),
    ("l1tex__t_sector_hit_rate.pct", "L1_hit_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]

TO_BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
TO_US = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarise(rep):
    h, units, data = raw(rep)
    out = []
    for r in data:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        rec = {"kernel": name}
        for k, short in KEYS:
            if k in h:
                v = r[h.index(k)].replace(",", "")
                u = units[h.index(k)]
                try:
                    x = float(v)
                except ValueError:
                    rec[short] = v
                    continue
                if short.startswith("dram_") and not short.endswith("%"):
                    x *= TO_BYTES.get(u, 1)
                if short == "time":
                    x *= TO_US.get(u, 1)
                rec[short] = x
        stalls = {c.split("smsp__pcsamp_warps_issue_stalled_")[1]: float(r[h.index(c)].replace(",", "") or 0)
                  for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not c.endswith("_not_issued")}
        tot = sum(stalls.values()) or 1
        rec["top_stalls"] = ", ".join(f"{k} {100*v/tot:.0f}%" for k, v in
                                      sorted(stalls.items(), key=lambda x: -x[1])[:4])
        out.append(rec)
    return out


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= h.index("Metric Value"):
            continue
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").split("<")[0]
        try:
            v = float(r[h.index("Metric Value")].replace(",", ""))
        except ValueError:
            continue
        agg[name][0] += 1
        agg[name][1] += v
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", nargs="*", default=[])
    ap.add_argument("--launches", nargs="*", default=[])
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic", default=None)
    ap.add_argument("--title", default="ncu summary")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    traffic = {}
    last_level = None
    for rep in a.rep:
        recs = summarise(rep)
        lines += [f"## `{rep.split('/')[-1]}` (`ncu --set full --clock-control none`)", "",
                  "| kernel | grid | regs | time us | DRAM rd MB | DRAM wr MB | DRAM % | L2 hit % | L1 hit % | warps active % | top stalls |",
                  "|---|---|---|---|---|---|---|---|---|---|---|"]
        for r in recs:
            lines.append(f"| {r['kernel']} | {r.get('grid','')} | {r.get('regs','')} | {r.get('time',0):.1f} | "
                         f"{r.get('dram_rd',0)/1e6:.1f} | {r.get('dram_wr',0)/1e6:.1f} | {r.get('dram_%',0):.1f} | "
                         f"{r.get('L2_hit_%',0):.1f} | {r.get('L1_hit_%',0):.1f} | {r.get('warps_active_%',0):.1f} | {r['top_stalls']} |")
            # one entry per LEVEL: the second kernel of a level (the CTA-unit
            # pass k_pull_heavy / k_heavy) adds to the entry its level opened
            base = r["kernel"].split("<")[0].split("::")[-1]
            byt = r.get("dram_rd", 0) + r.get("dram_wr", 0)
            key = {"k_pull": "VERTEX_PULL", "k_push_warp": "VERTEX_PUSH_WARP",
                   "k_edge": "EDGE_LIST", "k_push": "VERTEX_PUSH"}
            if base in ("k_pull_heavy", "k_heavy"):
                if last_level is not None:
                    traffic[last_level][-1] += byt
            elif base in key:
                last_level = key[base]
                traffic.setdefault(last_level, []).append(byt)
        lines.append("")
    for path in a.launches:
        agg = launches(path)
        tot = sum(v[1] for v in agg.values()) or 1
        lines += [f"## launch list `{path.split('/')[-1]}` (`--metrics gpu__time_duration.sum`, cold-cache, serialised)", "",
                  "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| {k or '(memcpy/memset)'} | {v[0]} | {v[1]/1e3:.1f} | {v[1]/tot:.3f} |")
        lines.append("")
    with open(a.out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    if a.traffic and traffic:
        with open(a.traffic, "w") as fh:
            json.dump({k: {"bytes_per_launch_mean": sum(v) / len(v), "launches": len(v),
                           "source": "ncu --set full of the launch-path kernels of each level (strategy kernel + its CTA-unit pass), tree-switched run of the bench roots"}
                       for k, v in traffic.items()}, fh, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
