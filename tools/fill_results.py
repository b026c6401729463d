"""Summarise a GPU evidence run (tools/gpu_r2_evidence.sh output dir) into markdown: the
BASELINE.md section-4 results table (bench lines + parity record) and the parity record table.
usage: python tools/fill_results.py gpurun_out/r2 > profiles/r02_results.md"""
import glob
import json
import os
import sys

D = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/r2"


def load(path):
    try:
        with open(path) as f:
            lines = [l for l in f.read().splitlines() if l.startswith("{")]
        return json.loads(lines[-1]) if lines else None
    except OSError:
        return None


rows = []
for path in sorted(glob.glob(os.path.join(D, "bench_c5*.json")) + glob.glob(os.path.join(D, "configs", "bench_*.json"))):
    b = load(path)
    if b:
        rows.append((os.path.basename(path)[6:-5], b))
par = []
pp = os.path.join(D, "parity_record.jsonl")
if os.path.exists(pp):
    par = [json.loads(l) for l in open(pp)]


def worst(case_prefix, kind):
    """worst L2 error over the recorded arrays of a parity case (states or gradients)"""
    keys = ("x", "v", "C", "F") if kind == "state" else ("dx0", "dv0", "dC0", "dF0", "dtheta")
    errs = [(r["l2_err"], r["array"], r["case"]) for r in par if r["case"].startswith(case_prefix) and r["array"] in keys]
    if not errs:
        return "--"
    e = max(errs)
    return f"{e[0]:.1e} ({e[1]}, {e[2]})"


PAR = {"c1a": "c1a", "c1b": "c1b", "c2": "c2@1024", "c2cl": "c2cl@256", "c3": "c3@512", "c3cl": "c3cl@96",
       "c3liquid": "c3liquid@176", "c4": "c4@128", "c5": "c5@64", "c5_k32": "c5@64"}
print("| config | particle-steps/s (fwd+bwd) | e2e | ms / iteration | k | dominant kernel: frac of HBM peak | "
      "step byte-model frac | A (active nodes / episode) | SM clock MHz | oracle fp64 (fp32) particle-steps/s, 1 core | "
      "state rel err (worst) | grad rel-L2 (worst) |")
print("|---" * 12 + "|")
for name, b in rows:
    r = b.get("roofline", {})
    cpu = b.get("cpu_baseline") or {}
    f32 = (cpu.get("f32_build") or {}).get("value")
    cpu_s = f"{cpu['value']:.3g}" + (f" ({f32:.3g})" if f32 else "") if cpu.get("value") else "--"
    cfg = b.get("config", {})
    print(f"| {name} | {b['value']:.4g} | {b['e2e']['value']:.4g} | {b['ms_per_step']:.1f} | {cfg.get('k_ckpt')} | "
          f"{r.get('kernel')} {r.get('frac', 0):.3f} | {r.get('step_frac', 0):.3f} | {r.get('active_nodes_per_episode', 0):.0f} | "
          f"{(b.get('clocks') or {}).get('sm_mhz')} | {cpu_s} | {worst(PAR.get(name, name), 'state')} | "
          f"{worst(PAR.get(name, name), 'grad')} |")
if par:
    print()
    print("| parity case | episode | array | L2 err | L2 gate | max err | max gate | oracle fp32 L2 | fallback gate used |")
    print("|---" * 9 + "|")
    for r in par:
        f32 = r.get("oracle_f32_l2")
        print(f"| {r['case']} | {r['episode']} | {r['array']} | {r['l2_err']:.2e} | {r['l2_gate']:.0e} | "
              f"{r['max_err']:.2e} | {r['max_gate']:.0e} | {'--' if f32 is None else f'{f32:.1e}'} | "
              f"{'yes' if r.get('fallback_used') else 'no'} |")
