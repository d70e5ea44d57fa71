"""Summarise an ncu --set full report: top SASS instructions by warp-stall
samples for one kernel (reads `ncu -i <rep> --page source --print-source sass`).

    python tools/ncu_hot.py <report.ncu-rep> <kernel-regex> [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr_i]
data = [r for r in rows[hdr_i + 1:] if len(r) == len(h) and r[0] != "Address"]
S = h.index("Warp Stall Sampling (All Samples)")
stalls = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(r[S] or 0) for r in data)
print(f"{len(data)} SASS lines, {tot} stall samples")
for idx, r in sorted(enumerate(data), key=lambda x: -int(x[1][S] or 0))[:top]:
    reasons = sorted(((int(r[i] or 0), h[i][6:]) for i in stalls), reverse=True)[:3]
    rs = " ".join(f"{n}:{v}" for v, n in reasons if v)
    print(f"{idx:5d} {int(r[S]):6d} {100*int(r[S])/max(tot,1):5.1f}%  {r[1].strip()[:60]:60s} {rs}")
