"""Per-kernel table from an ncu --set full report: time, instructions, occupancy, issue,
DRAM / L1 / L2 traffic and the top stall reasons.  Usage: python tools/ncu_kernel_table.py REP"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
col = {n: i for i, n in enumerate(h)}


def g(r, n, scale=1.0):
    try:
        return float(r[col[n]]) * scale
    except (KeyError, ValueError):
        return float("nan")


stall = [n for n in h if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued")]
print(f"{'kernel':22s} {'us':>7s} {'Minstr':>7s} {'warps%':>6s} {'issue%':>6s} {'regs':>4s} {'dramMB':>7s} "
      f"{'L1ldMB':>7s} {'L1stMB':>7s} {'smemWF':>7s} {'l1%':>5s} {'l2%':>5s}  stalls")
for r in rows[2:]:
    name = r[col["Kernel Name"]].split("::")[-1].split("(")[0]
    st = sorted(((g(r, n), n.replace("smsp__pcsamp_warps_issue_stalled_", "")) for n in stall), reverse=True)
    tot = sum(v for v, _ in st) or 1
    print(f"{name:22s} {g(r, 'gpu__time_duration.sum'):7.1f} {g(r, 'smsp__inst_executed.sum', 1e-6):7.2f} "
          f"{g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f} "
          f"{g(r, 'sm__inst_issued.avg.pct_of_peak_sustained_active'):6.1f} {g(r, 'launch__registers_per_thread'):4.0f} "
          f"{g(r, 'dram__bytes_read.sum') + g(r, 'dram__bytes_write.sum'):7.1f} "
          f"{g(r, 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 32e-6):7.1f} "
          f"{g(r, 'l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum', 32e-6):7.1f} "
          f"{g(r, 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 1e-6):7.2f} "
          f"{g(r, 'l1tex__throughput.avg.pct_of_peak_sustained_active'):5.1f} "
          f"{g(r, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):5.1f}  "
          + " ".join(f"{n}={100 * v / tot:.0f}" for v, n in st[:5]))
