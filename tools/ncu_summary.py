"""Print the headline metrics of an ncu report: python tools/ncu_summary.py rep.ncu-rep [...]"""
import csv, subprocess, sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "Eligible Warps Per Scheduler",
        "Active Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Dynamic Shared Memory Per Block", "Block Limit Shared Mem", "Block Limit Registers",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Grid Size", "Waves Per SM"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki, mi, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    print("==", rep, rows[1][ki][:60])
    seen = set()
    for r in rows[1:]:
        if r[mi] in WANT and r[mi] not in seen:
            seen.add(r[mi])
            print(f"  {r[mi]:40s} {r[vi]:>14s} {r[ui]}")
    # warp stall reasons (raw page)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) >= 3:
        hdr, vals = rr[0], rr[2]
        st = []
        for n, v in zip(hdr, vals):
            if n.startswith("smsp__average_warp_latency_issue_stalled_") and n.endswith(".ratio") or \
               (n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued")):
                try:
                    st.append((float(v.replace(",", "")), n))
                except ValueError:
                    pass
        for v, n in sorted(st, reverse=True)[:8]:
            print(f"  stall {n:70s} {v}")
        for n, v in zip(hdr, vals):
            if n in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                     "lts__t_bytes.sum", "l1tex__t_bytes.sum", "smsp__inst_executed.sum"):
                print(f"  {n:40s} {v}")
