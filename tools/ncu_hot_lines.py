"""Per-source-line instruction counts and stall samples of one kernel in an
ncu report (compiled with -lineinfo):  python tools/ncu_hot_lines.py rep kernel-regex [N]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-skip", str(int(sys.argv[4]) if len(sys.argv) > 4 else 0), "--launch-count", "1", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, recs = "", None, []
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0] and len(r) >= 8:   # a source line row (SASS rows have an empty first column)
        try:
            recs.append((float(r[4] or 0), float(r[7] or 0), fname, r[0], r[1].strip()[:90]))
        except ValueError:
            pass
tot_s = sum(x[0] for x in recs) or 1
tot_i = sum(x[1] for x in recs) or 1
print(f"total samples {tot_s:.0f}, warp instructions {tot_i / 1e6:.1f}M")
for s, i, f, line, src in sorted(recs, reverse=True)[:n]:
    print(f"{100 * s / tot_s:5.1f}% smp {100 * i / tot_i:5.1f}% inst  {f}:{line:5s} {src}")
