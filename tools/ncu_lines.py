"""Warp-stall samples per CUDA source line of one kernel in an ncu report.

    python tools/ncu_lines.py <report.ncu-rep> <kernel-regex> [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
cur_file = "?"
h = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        h = r
        continue
    if h is None or len(r) != len(h) or not r[0]:
        continue
    S = h.index("Warp Stall Sampling (All Samples)")
    E = h.index("Instructions Executed")
    try:
        v = int(r[S] or 0)
        ex = int(r[E] or 0)
    except ValueError:
        continue
    key = (cur_file, int(r[0]), r[1].strip()[:70])
    a = agg.setdefault(key, [0, 0, {}])
    a[0] += v
    a[1] += ex
    for i, name in enumerate(h):
        if name.startswith("stall_") and "(Not" not in name:
            try:
                a[2][name[6:]] = a[2].get(name[6:], 0) + int(float(r[i] or 0))
            except ValueError:
                pass
tot = sum(v[0] for v in agg.values())
print(f"{tot} stall samples")
for (f, ln, src), (v, ex, rs) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    why = " ".join(f"{k}={n}" for k, n in sorted(rs.items(), key=lambda x: -x[1])[:3] if n)
    print(f"{100 * v / max(tot, 1):5.1f}% {v:6d} {ex:8d}  {f}:{ln}  {src}  [{why}]")
