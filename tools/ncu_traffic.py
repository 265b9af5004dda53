"""DRAM traffic per launch of the bench's top kernels from one
`ncu --set full` capture -> profiles/traffic.json (read by bench.py for
roofline.traffic), plus a per-kernel summary line for profiles/.

    python tools/ncu_traffic.py <report.ncu-rep> <config> <summary-path-for-the-record>
"""

from __future__ import annotations

import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
# bench.py kernel keys -> the CUDA kernel that implements them
BENCH_NAMES = {"k_scatter": "k_scatter", "k_pool_fwd": "k_pool_ring"}
METRICS = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
           "launch__registers_per_thread", "lts__t_bytes.sum")


def read_raw(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "")
        rec = {"kernel": name.split("(")[0].replace("void ", "").split("<")[0].split("::")[-1],
               "full_name": name}
        for m in METRICS:
            try:
                rec[m] = float(d[m].replace(",", ""))
            except (KeyError, ValueError):
                rec[m] = None
        res.append(rec)
    return res


def main():
    rep, config, summary = sys.argv[1], sys.argv[2], sys.argv[3]
    recs = read_raw(rep)
    path = ROOT / "profiles" / "traffic.json"
    data = json.loads(path.read_text()) if path.exists() else {}
    cfg = data.setdefault(config, {})
    for bench_name, kname in BENCH_NAMES.items():
        hits = [r for r in recs if r["kernel"] == kname]
        if not hits:
            continue
        r = hits[0]
        rd, wr = r["dram__bytes_read.sum"], r["dram__bytes_write.sum"]
        cfg[bench_name] = {"kernel": kname, "dram_bytes": (rd or 0) + (wr or 0),
                           "dram_read": rd, "dram_write": wr,
                           "duration_ns_under_ncu": r["gpu__time_duration.sum"],
                           "registers": r["launch__registers_per_thread"],
                           "l2_bytes": r["lts__t_bytes.sum"], "source": summary}
    path.write_text(json.dumps(data, indent=1) + "\n")
    for r in recs:
        print(f"{r['kernel']:18s} dram {((r['dram__bytes_read.sum'] or 0) + (r['dram__bytes_write.sum'] or 0)) / 1e9:8.3f} GB"
              f"  time {(r['gpu__time_duration.sum'] or 0) / 1e6:7.3f} ms  regs {r['launch__registers_per_thread']}")


if __name__ == "__main__":
    main()
