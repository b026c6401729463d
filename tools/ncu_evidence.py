"""SURVEY 8(d) "required ncu evidence" per kernel from ncu --set full reports: DRAM bytes and
throughput, L2 atomic/reduction sectors (0 by design: no global atomics in the hot loops),
shared-memory bank conflicts vs wavefronts, FMA-pipe activity, achieved occupancy.
usage: python tools/ncu_evidence.py REP [REP ...]  -> markdown table"""
import csv
import re
import subprocess
import sys

COLS = [("DRAM MB", ["dram__bytes_read.sum", "dram__bytes_write.sum"], "MB"),
        ("DRAM % peak", ["dram__throughput.avg.pct_of_peak_sustained_elapsed"], None),
        ("L2 red+atom sectors", ["lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum"], None),
        ("smem bank conflicts", ["l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"], None),
        ("smem wavefronts", ["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"], None),
        ("FMA pipe % active", ["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"], None),
        ("achieved occupancy %", ["sm__warps_active.avg.pct_of_peak_sustained_active"], None)]


def val(row, col, units, name):
    if name not in col:
        alt = [c for c in col if c.endswith("." + name)]  # section-prefixed copies
        if not alt:
            return None
        name = alt[0]
    try:
        v = float(row[col[name]])
    except ValueError:
        return None
    u = units[col[name]]
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
    return v * scale if "byte" in u else v


print("| kernel | " + " | ".join(c[0] for c in COLS) + " |")
print("|---" * (len(COLS) + 1) + "|")
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    col = {n: i for i, n in enumerate(h)}
    seen = set()
    for r in rows[2:]:
        name = re.search(r"k_\w+?(?=[<(])", r[col["Kernel Name"]]).group(0)
        if name in seen:
            continue
        seen.add(name)
        cells = []
        for _, names, _u in COLS:
            vs = [val(r, col, units, n) for n in names]
            vs = [v for v in vs if v is not None]
            cells.append("n/a" if not vs else (f"{sum(vs):.1f}" if sum(vs) < 1e6 else f"{sum(vs):.3g}"))
        print(f"| {name} | " + " | ".join(cells) + " |")
