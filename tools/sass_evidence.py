"""Static SASS evidence of the staged kernels (cuobjdump, no GPU needed): per kernel, the count
of bulk-copy (UBLKCP = cp.async.bulk, TMA engine), mbarrier (SYNCS.*), CTA barrier (BAR),
global atomic/reduction (ATOMG/REDG/RED), shared-memory (LDS/STS/ATOMS) and FP (FFMA/FMUL/FADD)
instructions.  Usage: python tools/sass_evidence.py [LIB] > profiles/rNN_sass_ops.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1910_00935_b200/libmpm_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
kern, ops, full = None, {}, collections.defaultdict(collections.Counter)
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        dm = re.search(r"(k_[a-z_0-9]+?)(ILi([23])E)?E", name)
        kern = (dm.group(1) + (f"<{dm.group(3)}>" if dm.group(3) else "")) if dm else name
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if kern and m:
        full[kern][m.group(2) + (m.group(3) or "")] += 1
groups = {
    "UBLKCP (cp.async.bulk)": lambda o: o.startswith("UBLKCP"),
    "SYNCS (mbarrier)": lambda o: o.startswith("SYNCS"),
    "BAR": lambda o: o.startswith("BAR"),
    "GLOBAL_ATOM (ATOMG/REDG)": lambda o: o.split(".")[0] in ("ATOMG", "REDG", "RED", "ATOM"),
    "ATOMS (shared)": lambda o: o.startswith("ATOMS"),
    "LDS": lambda o: o.split(".")[0] == "LDS",
    "STS": lambda o: o.split(".")[0] == "STS",
    "LDG": lambda o: o.split(".")[0] == "LDG",
    "STG": lambda o: o.split(".")[0] == "STG",
    "FP32 (FFMA/FMUL/FADD)": lambda o: o.split(".")[0] in ("FFMA", "FMUL", "FADD"),
    "LDL/STL (spills)": lambda o: o.split(".")[0] in ("LDL", "STL"),
}
print(f"# static SASS op counts per kernel ({lib}; cuobjdump -sass, sm_100a)")
print("kernel".ljust(26) + "".join(g.split(" ")[0][:11].ljust(12) for g in groups))
for k in sorted(full):
    c = full[k]
    row = [sum(n for o, n in c.items() if f(o)) for f in groups.values()]
    print(k.ljust(26) + "".join(str(x).ljust(12) for x in row))
print("\n# distinct SYNCS / UBLKCP forms")
for k in sorted(full):
    forms = sorted(o for o in full[k] if o.startswith(("SYNCS", "UBLKCP")))
    if forms:
        print(f"{k}: " + ", ".join(f"{o} x{full[k][o]}" for o in forms))
