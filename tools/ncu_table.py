"""One line per captured launch of an ncu report: time, DRAM bytes and
bandwidth, L2 hit rate, registers, occupancy, issue activity, grid, plus the
top warp-stall reasons.   python tools/ncu_table.py rep.ncu-rep"""
import csv
import subprocess
import sys

W = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
     "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ix = {w: h.index(w) for w in W if w in h}
    stalls = [(i, n) for i, n in enumerate(h) if n.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not n.endswith("_not_issued")]
    print(f"== {rep}")
    for r in rows[2:]:
        v = {w: float(r[i].replace(",", "") or 0) for w, i in ix.items()}
        t = v["gpu__time_duration.sum"] / 1e6
        rd, wr = v["dram__bytes_read.sum"] / 1e9, v["dram__bytes_write.sum"] / 1e9
        name = r[h.index("Kernel Name")].replace("void ", "").split("(")[0][:34]
        print(f"{name:34s} {t:7.3f} ms  dram rd {rd:6.3f} wr {wr:6.3f} GB = {(rd + wr) / t:5.2f} TB/s"
              f"  L2hit {v.get('lts__t_sector_hit_rate.pct', 0):5.1f}%  regs {v['launch__registers_per_thread']:.0f}"
              f"  occ {v['sm__warps_active.avg.pct_of_peak_sustained_active']:5.1f}%"
              f"  issue {v['smsp__issue_active.avg.pct_of_peak_sustained_active']:5.1f}%"
              f"  grid {v['launch__grid_size']:.0f}  inst {v.get('smsp__inst_executed.sum', 0) / 1e6:.0f}M")
        st = sorted(((float(r[i].replace(",", "") or 0), n.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                     for i, n in stalls), reverse=True)[:4]
        print("    stalls: " + ", ".join(f"{n} {c:.0f}" for c, n in st))
