"""Summarise an ncu --csv launch list (one step): per-kernel launches, time and DRAM bytes.

  python tools/ncu_summarize.py gpurun_out/step_tf32.csv tf32 [profiles/ncu_traffic.json] [profiles/x.md]
Merges {precision: {kernel: {...}}} into the JSON file and writes a markdown table.
"""
import csv, io, json, os, sys
from collections import OrderedDict

src, prec = sys.argv[1], sys.argv[2]
out_json = sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_traffic.json"
out_md = sys.argv[4] if len(sys.argv) > 4 else None
txt = open(src).read()
txt = txt[txt.index('"ID"'):]
rows = list(csv.DictReader(io.StringIO(txt)))
per = OrderedDict()
for r in rows:
    name = r["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0].strip()
    launch = (r["ID"], name)
    d = per.setdefault(launch, {"name": name})
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
             "ns": 1e-3, "us": 1, "ms": 1e3}.get(unit, 1)
    d[r["Metric Name"]] = v * scale
agg = OrderedDict()
for (_, name), d in per.items():
    a = agg.setdefault(name, {"launches": 0, "gpu_time_us": 0.0, "dram_bytes": 0.0})
    a["launches"] += 1
    a["gpu_time_us"] += d.get("gpu__time_duration.sum", 0.0)
    a["dram_bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot = sum(a["gpu_time_us"] for a in agg.values())
res = {}
for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["gpu_time_us"]):
    res[name] = {"launches": a["launches"], "gpu_time_us": a["gpu_time_us"], "share": a["gpu_time_us"] / tot,
                 "dram_bytes_per_launch": a["dram_bytes"] / a["launches"],
                 "dram_gbs": a["dram_bytes"] / (a["gpu_time_us"] * 1e-6) / 1e9 if a["gpu_time_us"] else 0.0}
allj = {}
if os.path.exists(out_json):
    allj = json.load(open(out_json))
allj[prec] = res
allj.setdefault("_note", "ncu --profile-from-start off over one training step (tools/ncu_step.py), cold-cache "
                "serialised replays: dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged per kernel")
json.dump(allj, open(out_json, "w"), indent=1)
lines = [f"| kernel | launches | ncu time (us) | share | DRAM bytes/launch | DRAM GB/s |", "|---|---|---|---|---|---|"]
for name, a in res.items():
    lines.append(f"| {name} | {a['launches']} | {a['gpu_time_us']:.1f} | {a['share']*100:.1f}% | "
                 f"{a['dram_bytes_per_launch']/1e6:.3f} MB | {a['dram_gbs']:.0f} |")
lines.append(f"| total | {sum(a['launches'] for a in res.values())} | {tot:.1f} | | | |")
md = "\n".join(lines)
print(md)
if out_md:
    open(out_md, "w").write(md + "\n")
