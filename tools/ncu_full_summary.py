"""Markdown summary of one `ncu --set full` capture (.ncu-rep): per launch, duration, grid,
registers, DRAM bytes, SM / tensor-pipe / DRAM utilisation and the top warp-stall reasons.

  python tools/ncu_full_summary.py gpurun_out/prof_rowgemm.ncu-rep "title" >> profiles/x.md
"""
import csv
import io
import subprocess
import sys

COLS = [
    ("us", "gpu__time_duration.sum"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("regs", "launch__registers_per_thread"),
    ("DRAM rd", "dram__bytes_read.sum"),
    ("DRAM wr", "dram__bytes_write.sum"),
    ("SM %", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("DRAM %", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor pipe %", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
]
STALL = "smsp__average_warps_issue_stalled_"


def main():
    rep, title = sys.argv[1], sys.argv[2]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u, data = rows[0], rows[1], rows[2:]
    ix = {k: i for i, k in enumerate(h)}
    print(f"### {title}\n")
    print(f"`{rep.split('/')[-1]}` — `ncu --set full --clock-control none`, {len(data)} launches; "
          f"kernel `{data[0][ix['Kernel Name']].split('(')[0]}`.\n")
    cols = [(n, k) for n, k in COLS if k in ix]
    print("| # | " + " | ".join(f"{n} ({u[ix[k]]})" if u[ix[k]] else n for n, k in cols) + " | top stalls (warps per issue) |")
    print("|---" * (len(cols) + 2) + "|")
    stalls = [k for k in h if k.startswith(STALL) and k.endswith("_per_issue_active.ratio")]
    for j, r in enumerate(data):
        st = sorted(((float(r[ix[k]] or 0), k[len(STALL):-len("_per_issue_active.ratio")]) for k in stalls), reverse=True)[:3]
        vals = []
        for _, k in cols:
            v = r[ix[k]]
            try:
                f = float(v.replace(",", ""))
                v = f"{f:.1f}" if f != int(f) else str(int(f))
            except ValueError:
                pass
            vals.append(v)
        print(f"| {j} | " + " | ".join(vals) + " | " + ", ".join(f"{n} {x:.2f}" for x, n in st) + " |")
    print()


if __name__ == "__main__":
    main()
