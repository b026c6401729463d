"""Summarise an ncu source page per CUDA source line: stall samples and executed warp
instructions, hottest lines first.  Usage: python tools/ncu_line_summary.py REP KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
by_instr = len(sys.argv) > 4 and sys.argv[4] == "instr"  # sort by executed instructions
# (ncu prints this page only into a pipe; regexes must avoid '<')
out = subprocess.run(f"ncu -i {rep} --page source --csv --print-source cuda,sass -k regex:{kern} 2>&1 | cat",
                     shell=True, capture_output=True, text=True).stdout
fname, hdr, stats = "?", None, []
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].rsplit("/", 1)[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or not row[0] or len(row) < len(hdr):
        continue
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iE = hdr.index("Instructions Executed")
    try:
        s, e = int(float(row[iS] or 0)), int(float(row[iE] or 0))
    except ValueError:  # SASS rows and '-' cells
        continue
    stats.append((s, e, f"{fname}:{row[0]}", row[1].strip()[:90]))
merged = {}
for s_, e_, where, src in stats:  # several launches of the kernel: merge per line
    m = merged.setdefault(where, [0, 0, src])
    m[0] += s_
    m[1] += e_
stats = [(v[0], v[1], k, v[2]) for k, v in merged.items()]
tot_s = sum(s for s, *_ in stats) or 1
tot_e = sum(e for _, e, *_ in stats) or 1
print(f"stall samples {tot_s}, warp-instr {tot_e}")
key = (lambda t: t[1]) if by_instr else (lambda t: t[0])
for s, e, where, src in sorted(stats, key=key, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% {100*e/tot_e:5.1f}%  {where:22s} {src}")
