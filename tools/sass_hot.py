"""Hot SASS blocks of an ncu report: python tools/sass_hot.py rep.ncu-rep [section] [top]
Groups consecutive instructions with equal execution counts (basic blocks)."""
import csv, subprocess, sys

rep = sys.argv[1]
sec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 14
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
s0 = starts[sec]
s1 = starts[sec + 1] if sec + 1 < len(starts) else len(rows)
print(rows[s0][1])
h = rows[s0 + 1]
d = [r for r in rows[s0 + 2:s1] if len(r) == len(h)]
ie = h.index("Instructions Executed")
ws = h.index("Warp Stall Sampling (All Samples)")
blocks = []
for r in d:
    c = float(r[ie] or 0)
    op = r[1].split()[0] if r[1] else ""
    if op.startswith("@"):
        op = r[1].split()[1]
    if blocks and blocks[-1][1] == c:
        blocks[-1][2] += 1
        blocks[-1][3].append(op)
        blocks[-1][4] += float(r[ws] or 0)
    else:
        blocks.append([r[0], c, 1, [op], float(r[ws] or 0)])
tot = sum(b[1] * b[2] for b in blocks)
stot = sum(b[4] for b in blocks) or 1
print(f"warp instructions {tot:.3e}")
for b in sorted(blocks, key=lambda b: -b[1] * b[2])[:top]:
    print(f"{b[0][-5:]} {b[1]/1e6:7.2f}M x{b[2]:3d} = {b[1]*b[2]/tot*100:5.1f}% stall {b[4]/stot*100:5.1f}%  "
          + " ".join(b[3][:16]))
