"""Per-source-line instruction / divergence / stall-sample totals of one
kernel in an ncu report (SASS page + nvdisasm line map of the same build).

    python tools/ncu_lines.py report.ncu-rep <mangled kernel> [cubin [top [samples]]]
"""
import collections, csv, re, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
cubin = sys.argv[3] if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(raw))
hdr = rows[1]
data = rows[2:]
ia, ie, it, ism = (hdr.index(k) for k in ("Address", "Instructions Executed",
                                           "Thread Instructions Executed",
                                           "Warp Stall Sampling (All Samples)"))
if cubin is None:
    subprocess.run("rm -rf /tmp/ncu_lines_cub && mkdir -p /tmp/ncu_lines_cub && cd /tmp/ncu_lines_cub && "
                   "cuobjdump -xelf all /root/repo/paper_1708_01159_b200/libabfs.so >/dev/null",
                   shell=True, check=True)
    cubin = "/tmp/ncu_lines_cub/engine.sm_100a.cubin"
lines = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.split("\n")
start = [i for i, l in enumerate(lines) if l.startswith(".text." + kern + ":")][0]
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith(".text.")), len(lines))
amap, cur = {}, None
for l in lines[start:end]:
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        amap[int(m.group(1), 16)] = cur
base = int(data[0][ia], 16)
by = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
tot = [0.0, 0.0, 0.0]
for r in data:
    try:
        a = int(r[ia], 16) - base
    except ValueError:
        continue
    vals = [float(r[ie] or 0), float(r[it] or 0), float(r[ism] or 0)]
    b = by[amap.get(a)]
    for k in range(3):
        b[k] += vals[k]
        tot[k] += vals[k]
print(f"warp inst {tot[0]/1e6:.1f}M thread inst {tot[1]/1e6:.1f}M avg threads/inst "
      f"{tot[1]/tot[0]:.1f} stall samples {tot[2]:.0f}")
key = 2 if len(sys.argv) > 5 and sys.argv[5] == "samples" else 0   # sort by stall samples
for ln, b in sorted(by.items(), key=lambda x: -x[1][key])[:int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    print(f"{ln}  inst {b[0]/1e6:6.2f}M ({100*b[0]/tot[0]:4.1f}%)  threads/inst {b[1]/max(b[0],1):4.1f}"
          f"  samples {100*b[2]/tot[2]:4.1f}% ({b[2]:.0f})")
