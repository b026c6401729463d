"""Summarise ptxas -v output in paper_1910_00935_b200/build.log: registers, spills, smem per kernel."""
import re
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_1910_00935_b200/build.log").read().splitlines()
name = None
props = {}
for line in log:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        name = m.group(1)
        props[name] = {}
        continue
    if name is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        props[name]["stack"], props[name]["spill_st"], props[name]["spill_ld"] = map(int, m.groups())
    m = re.search(r"Used (\d+) registers", line)
    if m:
        props[name]["regs"] = int(m.group(1))
        sm = re.search(r"(\d+) bytes smem", line)
        props[name]["smem"] = int(sm.group(1)) if sm else 0
for n, p in props.items():
    m = re.search(r"(k_[a-z0-9_]+?)(ILi(\d)E)?E", n)
    short = (m.group(1) + (f"<{m.group(3)}>" if m.group(3) else "")) if m else n
    print(f"{short:28s} regs={p.get('regs')} stack={p.get('stack')} spill={p.get('spill_st')}/{p.get('spill_ld')} smem={p.get('smem')}")
