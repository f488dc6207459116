"""Summarise ptxas -v logs: registers, stack, spills per kernel (flags spills)."""
import glob
import re
import subprocess
import sys

logs = sys.argv[1:] or sorted(glob.glob("paper_1810_10197_b200/_build/*.ptxas.log"))
pat_fn = re.compile(r"Compiling entry function '(\S+)'")
pat_sp = re.compile(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads")
pat_rg = re.compile(r"Used (\d+) registers")
for log in logs:
    fn = sp = None
    for line in open(log):
        m = pat_fn.search(line)
        if m:
            fn, sp = m.group(1), None
            continue
        m = pat_sp.search(line)
        if m and fn:
            sp = tuple(int(x) for x in m.groups())
            continue
        m = pat_rg.search(line)
        if m and fn:
            name = subprocess.run(["c++filt"], input=fn, capture_output=True, text=True).stdout.strip()
            flag = "  <-- SPILL" if sp and (sp[1] or sp[2]) else ""
            print(f"{int(m.group(1)):4d} regs  stack {sp[0] if sp else '?':>5}  spill {sp[1] if sp else '?':>5}/"
                  f"{sp[2] if sp else '?':<5} {name[:110]}{flag}")
            fn = None
