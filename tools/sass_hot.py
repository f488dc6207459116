"""Instruction mix + stall hot spots from `ncu --page source --print-source sass --csv` output."""
import collections
import csv
import sys


def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return None


rows = list(csv.reader(open(sys.argv[1])))
hdr_i = [i for i, r in enumerate(rows) if "Source" in r and "Address" in r]
h = rows[hdr_i[0]]
si, ni, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
ops, opsS = collections.Counter(), collections.Counter()
recs = []
tot_s = tot_e = 0.0
for r in rows[hdr_i[0] + 1:]:
    if len(r) <= ei:
        continue
    s, e = num(r[ni]), num(r[ei])
    if s is None or e is None:
        continue
    toks = r[si].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    ops[op] += e
    opsS[op] += s
    tot_s += s
    tot_e += e
    recs.append((s, r[0], r[si][:70]))
print("warp-instructions executed", tot_e)
for op, e in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 22):
    print(f"{op:10s} {e / tot_e * 100:5.1f}% instr  {opsS[op] / max(tot_s, 1) * 100:5.1f}% stall-samples")
print("top stall instructions:")
for s, a, src in sorted(recs, reverse=True)[:20]:
    print(f"{s / max(tot_s, 1) * 100:5.2f}% {a} {src}")
