"""Per-source-line instruction/stall view of an `ncu --page source --print-source
cuda,sass` CSV (tools/gpu_round.sh): python tools/src_top.py file.csv [n] [warp_steps]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
norm = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
cur = None
lines = {}
sass = []
line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "" and len(r) > 8:
        try:
            lines[(cur, int(r[0]))] = (r[1][:100], int(r[7] or 0), int(r[4] or 0))
            line = (cur, int(r[0]))
        except ValueError:
            pass
    elif len(r) > 8 and r[2].startswith("0x"):
        sass.append((line, r[3].strip(), int(r[4] or 0), int(r[7] or 0)))
ti = sum(v[1] for v in lines.values())
ts = sum(v[2] for v in lines.values()) or 1
print(f"instructions {ti}  stall samples {ts}" + (f"  per unit {ti / norm:.1f}" if norm else ""))
for k, v in sorted(lines.items(), key=lambda kv: -kv[1][1])[:n]:
    per = f"{v[1] / norm:7.1f}" if norm else f"{100 * v[1] / ti:6.1f}%"
    print(f"{k[0][:12]:12s}{k[1]:5d} {per} st{100 * v[2] / ts:5.1f}%  {v[0]}")
print("-- top stall SASS --")
for s in sorted(sass, key=lambda s: -s[2])[:12]:
    print(f"{100 * s[2] / ts:5.1f}% L{s[0][1] if s[0] else '?':>5} {s[1][:70]}")
