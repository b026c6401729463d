"""Build an A/B variant of libmpm_b200.so with extra nvcc flags into variants/NAME.so.
usage: python tools/build_variant.py NAME [-DKNOB=V ...]   (run on the GPU box with tools/ab.sh)"""
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1910_00935_b200 import build as B  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
out = os.path.join(ROOT, "variants", name + ".so")
B.build(force=True, extra=extra, out=out)
log = open(out + ".log").read()
for m in re.finditer(r"Compiling entry function '(\w+)' for 'sm_100a'\n(.*?)\n(.*?)\n", log):
    if "ILi3E" in m.group(1) and re.search(r"k_(p2g|g2p)", m.group(1)):
        fn = re.search(r"k_\w+?(?=I)", m.group(1)).group(0)
        print(f"{name:18s} {fn:12s} {m.group(2).split(':')[-1].strip()[:70]} | {m.group(3).split(':')[-1].strip()[:60]}")
