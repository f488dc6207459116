"""Top stalled SASS instructions of one kernel in an .ncu-rep (source page, sass view).

    python tools/sass_stalls.py <rep> <kernel-regex> [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}",
                      "--launch-skip", str(skip), "--launch-count", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
S = h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") or "Stall" in c and i > S + 1]
# per-reason columns are named like "smsp__pcsamp_warps_issue_stalled_*" or short names; keep numeric ones after '# Samples'
reason_cols = [(i, c) for i, c in enumerate(h) if i > h.index("# Samples") and c not in (
    "Instructions Executed", "Thread Instructions Executed", "Predicated-On Thread Instructions Executed",
    "Avg. Threads Executed", "Avg. Predicated-On Threads Executed", "Divergent Branches", "Address Space",
    "Access Operation", "Access Size") and not c.startswith("L1") and not c.startswith("L2")]
rows = [rows[0]] + [r for r in rows[1:] if r and r[0].startswith("0x")]
tot = sum(float(r[S] or 0) for r in rows[1:])
print(lines[0][:150])
print(f"total samples {tot:.0f}")
byop = defaultdict(float)
for r in rows[1:]:
    op = r[src].split()[0] if r[src].split() else "?"
    if op.startswith("@"):
        op = r[src].split()[1]
    byop[op.split(".")[0]] += float(r[S] or 0)
print("by opcode:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in sorted(byop.items(), key=lambda x: -x[1])[:14]))
ranked = sorted(rows[1:], key=lambda r: -float(r[S] or 0))[:top]
for r in ranked:
    reasons = sorted(((float(r[i] or 0) if r[i].replace('.', '', 1).isdigit() else 0, c) for i, c in reason_cols), reverse=True)[:3]
    rs = " ".join(f"{c}={v:.0f}" for v, c in reasons if v > 0)
    print(f"{float(r[S]) / tot * 100:5.1f}%  {r[0][-5:]}  {r[src].strip()[:60]:60s} {rs}")
