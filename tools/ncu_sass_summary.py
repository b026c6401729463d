"""Summarise an ncu SASS source page: executed instructions and stall samples per opcode,
and the hottest instruction windows.  Usage: python tools/ncu_sass_summary.py REP KERNEL_REGEX"""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
# (ncu prints this page only into a pipe; regexes must avoid '<')
out = subprocess.run(f"ncu -i {rep} --page source --csv --print-source sass -k regex:{kern} 2>&1 | cat",
                     shell=True, capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"Kernel Name"')), len(lines))
rows = list(csv.reader(lines[start:end]))
hdr = rows[0]
iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
ops = collections.defaultdict(lambda: [0, 0])
seq = []
for r in rows[1:]:
    if len(r) < len(hdr):
        continue
    src = r[1].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    s, e = int(r[iS] or 0), int(float(r[iE] or 0))
    ops[op][0] += e
    ops[op][1] += s
    seq.append((r[0], src, s, e))
tot_e = sum(v[0] for v in ops.values())
tot_s = sum(v[1] for v in ops.values())
print(f"total executed warp-instr {tot_e}, stall samples {tot_s}")
for op, (e, s) in sorted(ops.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {op:10s} exec {e:10d} ({100*e/tot_e:5.1f}%)  samples {s:7d} ({100*s/tot_s:5.1f}%)")
# hottest 40-instruction windows
W = 40
best = sorted(((sum(x[2] for x in seq[i:i+W]), i) for i in range(0, max(1, len(seq)-W), W)), reverse=True)[:4]
for s, i in best:
    print(f"--- window @{i} samples {s}")
    for a, src, ss, ee in seq[i:i+W]:
        if ss > tot_s * 0.002:
            print(f"    {ss:6d} {ee:9d}  {src[:90]}")
