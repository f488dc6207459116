"""Summarise an .ncu-rep: per kernel duration, DRAM bytes, throughputs, occupancy, top stalls."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active"]
idx = {w: h.index(w) for w in want if w in h}
stall = [(i, c) for i, c in enumerate(h) if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")]
units = rows[1]
for r in rows[2:]:
    print("==", r[idx["Kernel Name"]][:110])
    for w in want[1:]:
        if w in idx:
            print(f"   {w:70s} {r[idx[w]]:>16s} {units[idx[w]]}")
    st = sorted(((float(r[i] or 0), c.replace('smsp__pcsamp_warps_issue_stalled_', '')) for i, c in stall), reverse=True)[:6]
    tot = sum(float(r[i] or 0) for i, _ in stall)
    print("   top stalls:", ", ".join(f"{n} {v / tot * 100:.0f}%" for v, n in st))
