"""Markdown summary of an ncu launch list (`--metrics gpu__time_duration.sum --csv --log-file X`):
launches, summed time and share per kernel.

  python tools/ncu_launch_summary.py gpurun_out/launches_bench.csv "title" "command" > profiles/x.md
"""
import csv
import io
import sys
from collections import defaultdict

SCALE = {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}


def main():
    path, title, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        n = r["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0].strip()
        agg[n][0] += 1
        agg[n][1] += float(r["Metric Value"].replace(",", "")) * SCALE[r["Metric Unit"]]
    tot = sum(v[1] for v in agg.values())
    print(f"# {title}\n")
    print(f"`{cmd}`: {len(rows)} launches captured. Cold-cache serialised per-launch times; the kernel "
          "SHARE is what bench.py's live CUDA-event roofline must agree with.\n")
    print("| kernel | launches | ncu time (us) | share |\n|---|---|---|---|")
    for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {n} | {c} | {t:.1f} | {100 * t / tot:.1f}% |")
    print(f"| total | {len(rows)} | {tot:.1f} | |")


if __name__ == "__main__":
    main()
