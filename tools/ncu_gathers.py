"""Per-source-line global-memory sector efficiency of one kernel in an ncu
report: for every SASS load/store/atomic, ncu's L1 tag requests, L2
theoretical sectors (actual / ideal / excessive) and instructions executed,
attributed through the inlining chain (`nvdisasm -gi`) to our own source
line and its caller.  sectors/request = 32-byte sectors fetched per warp-wide
request (4 = a coalesced 4-byte-per-lane load; 32 = fully scattered).

    python tools/ncu_gathers.py report.ncu-rep <mangled kernel> [--top N] [--md out.md]
"""
import argparse
import collections
import csv
import re
import subprocess
import tempfile

OWN = ("bfs_kernels.cuh", "megakernel.cuh", "pull2.cuh", "engine.cu", "partition.cu", "launch.cuh")


def line_map(cubin, kern):
    out = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout.split("\n")
    start = next(i for i, ln in enumerate(out) if ln.startswith(".text." + kern + ":"))
    end = next((i for i in range(start + 1, len(out)) if out[i].startswith(".text.")), len(out))
    amap, cur, group = {}, None, []
    pat = re.compile(r'File "([^"]+)", line (\d+)')
    for ln in out[start:end]:
        if "//## File" in ln:
            # a group of //## lines precedes each block: (callee, caller)
            # pairs, innermost first
            group += [(f.split("/")[-1], int(n)) for f, n in pat.findall(ln)]
            continue
        if group:
            frames = list(dict.fromkeys(group))
            own = [fr for fr in frames if fr[0] in OWN]
            cur = tuple(own[:2]) if own else tuple(frames[:1])
            group = []
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m:
            amap[int(m.group(1), 16)] = cur
    return amap


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("kernel")
    ap.add_argument("--so", default="/root/repo/paper_1708_01159_b200/libabfs.so")
    ap.add_argument("--cubin", default="engine.sm_100a.cubin")
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--md", default=None)
    a = ap.parse_args()
    tmp = tempfile.mkdtemp()
    subprocess.run(f"cd {tmp} && cuobjdump -xelf all {a.so} > /dev/null", shell=True, check=True)
    amap = line_map(f"{tmp}/{a.cubin}", a.kernel)
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    col = {k: hdr.index(k) for k in ("Address", "Source", "Instructions Executed", "Access Operation",
                                     "L1 Tag Requests Global", "L2 Theoretical Sectors Global",
                                     "L2 Theoretical Sectors Global Ideal",
                                     "Warp Stall Sampling (All Samples)")}
    base = int(data[0][col["Address"]], 16)
    agg = collections.defaultdict(lambda: collections.Counter())
    tot = collections.Counter()

    def num(r, k):
        try:
            return float(r[col[k]].replace(",", ""))
        except ValueError:
            return 0.0
    for r in data:
        addr = int(r[col["Address"]], 16) - base
        key = amap.get(addr)
        sass = r[col["Source"]].strip()
        op = sass.split()[0] if sass else "?"
        if op.startswith("@"):
            op = sass.split()[1]
        req = num(r, "L1 Tag Requests Global")
        sec = num(r, "L2 Theoretical Sectors Global")
        ideal = num(r, "L2 Theoretical Sectors Global Ideal")
        samples = num(r, "Warp Stall Sampling (All Samples)")
        tot["samples"] += samples
        tot["inst"] += num(r, "Instructions Executed")
        if req == 0 and sec == 0:
            if key:
                agg[(key, "-")]["samples"] += samples
            continue
        k = (key, op.split(".")[0])
        c = agg[k]
        c["req"] += req
        c["sec"] += sec
        c["ideal"] += ideal
        c["samples"] += samples
        c["inst"] += num(r, "Instructions Executed")
        tot["req"] += req
        tot["sec"] += sec
    items = sorted(((k, v) for k, v in agg.items() if v["req"]), key=lambda kv: -kv[1]["sec"])
    lines = [f"# Global-memory sector efficiency per source line: `{a.kernel}`", "",
             f"report `{a.rep}`; totals: {tot['req']:.0f} requests, {tot['sec']:.0f} L2 sectors "
             f"({tot['sec'] * 32 / 1e9:.3f} GB), {tot['sec'] / max(1, tot['req']):.2f} sectors/request, "
             f"{tot['inst']:.0f} warp instructions", "",
             "| line (inlined at) | op | requests | L2 sectors | sectors/req | ideal sectors | excess % | stall samples % |",
             "|---|---|---|---|---|---|---|---|"]
    for (key, op), v in items[:a.top]:
        where = " <- ".join(f"{f}:{n}" for f, n in key) if key else "?"
        exc = 100.0 * (v["sec"] - v["ideal"]) / v["sec"] if v["sec"] else 0.0
        lines.append(f"| {where} | {op} | {v['req']:.0f} | {v['sec']:.0f} | {v['sec'] / v['req']:.2f} | "
                     f"{v['ideal']:.0f} | {exc:.1f} | {100 * v['samples'] / max(1, tot['samples']):.1f} |")
    text = "\n".join(lines)
    print(text)
    if a.md:
        with open(a.md, "w") as fh:
            fh.write(text + "\n")


if __name__ == "__main__":
    main()
