"""Attribute ncu warp-stall samples (SASS view) to CUDA source lines via nvdisasm line info.

  python tools/sass_lines.py report.ncu-rep KERNEL_SUBSTR CUBIN [launch_index] [top]
"""
import csv, io, re, subprocess, sys
from collections import defaultdict

rep, kname, cubin = sys.argv[1], sys.argv[2], sys.argv[3]
li = int(sys.argv[4]) if len(sys.argv) > 4 else 0
top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
syms = subprocess.run(["cuobjdump", "-symbols", cubin], capture_output=True, text=True).stdout
mang = [w for w in re.findall(r"\S+", syms) if kname in w][0]
dis_all = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
start = [i for i, ln in enumerate(dis_all) if ".text." + mang in ln and "section" in ln][0]
end = next((i for i in range(start + 1, len(dis_all)) if ".section" in dis_all[i] and ".text." in dis_all[i]), len(dis_all))
line_of, cur = {}, None
for ln in dis_all[start:end]:
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", kname,
                      "--launch-skip", str(li), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hdr_i]
data = [r for r in rows[hdr_i + 1:] if len(r) == len(h)]
iS = h.index("Warp Stall Sampling (All Samples)")
base = int(data[0][0], 16)
agg = defaultdict(int)
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ri = [h.index(c) for c in reasons]
why = defaultdict(lambda: defaultdict(int))
tot = 0
num = lambda x: int(x) if x.strip().isdigit() else 0
for r in data:
    s = num(r[iS])
    tot += s
    key = line_of.get(int(r[0], 16) - base, ("?", 0))
    agg[key] += s
    for c, i in zip(reasons, ri):
        why[key][c] += num(r[i])
src = {}
for f in set(k[0] for k in agg):
    try:
        src[f] = open(f"/root/repo/paper_2412_20796_b200/csrc/{f}").read().splitlines()
    except Exception:
        src[f] = []
print("total samples", tot)
for (f, l), s in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    code = src.get(f, [])[l - 1].strip()[:90] if 0 < l <= len(src.get(f, [])) else ""
    w = sorted(why[(f, l)].items(), key=lambda kv: -kv[1])[:3]
    ws = " ".join(f"{k[6:]}={v}" for k, v in w if v)
    print(f"{100.0 * s / max(tot, 1):5.1f}%  {f}:{l:<5d} {code[:70]:70s} [{ws}]")
