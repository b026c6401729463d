#!/usr/bin/env python
"""Benchmark: fwd+bwd particle-steps/s of the differentiable MLS-MPM hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

One bench "step" = one optimisation iteration of the whole hot path on one
batch of synthetic input: set_state -> forward(T) (checkpointed tape) -> loss
-> backward(T) -> grads -> NCCL all-reduce of the shared-parameter gradient
(N > 1).  value = particles x time steps x K (all ranks) / max-over-ranks
device time.  Default workload: C5 (BASELINE.json configs[4]: 1,061,208
particles, 128^3 grid, 2,048 steps, k = 32), one episode per GPU (weak scaling).

--impl reference times the CPU oracle (oracle/, the only reference this paper
has) on the host cores: each step is a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd particle-steps/s (2D/3D MLS-MPM) at 1/2/4/8 B200; % HBM roofline"
UNIT = "particle-steps/s"


# ------------------------------------------------------------------ helpers
def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def _workload(name: str, world: int, rank: int = 0):
    """config, this rank's episode indices, scaling kind.  C4: 64 episodes split over
    the ranks (strong scaling); others: one episode per rank (weak scaling)."""
    from paper_1910_00935_b200 import workloads as W
    from paper_1910_00935_b200.dist import episode_shard
    p = W.config(name)
    if os.environ.get("BENCH_HORIZON"):  # experiments only (e.g. k = 1 vs 2 at a horizon where k = 1 fits)
        p["steps"] = int(os.environ["BENCH_HORIZON"])
    if name == "c4":
        return p, episode_shard(int(p["episodes"]), rank, world), "strong"
    return p, range(rank, rank + 1), "weak"


def _describe(p, n_particles, episodes, world, k):
    shape = {"cube3d": "3D elastic cube", "robot3d": "3D robot (16 muscles)",
             "robot3d_liquid": "3D robot (16 muscles) + liquid block",
             "robot2d": "2D robot (4 muscles)", "block2d": "2D elastic block"}[p["shape"]]
    return {"workload": f"{p['name']}: {shape}, {n_particles:,} particles x {episodes} episode(s)/GPU, "
                        f"{p['n_grid']}^{p['dim']} grid, {p['steps']} steps, checkpoint every {k}",
            "config_index": {"c1a": 0, "c1b": 0, "c2": 1, "c2cl": 1, "c3": 2, "c3cl": 2, "c3liquid": 2, "c4": 3, "c5": 4}[p["name"]],
            "controller": ("closed loop (R22)" if p.get("closed_loop") else "open loop") if p.get("n_act") else "none",
            "dim": p["dim"], "particles_per_episode": n_particles, "episodes_per_gpu": episodes,
            "episodes_total": episodes * world, "n_grid": p["n_grid"], "time_steps": p["steps"],
            "k_ckpt": k, "model": p["model"], "parallelism": f"episodes x{world} (dp{world})",
            "l2": "inputs larger than L2 (per-step state stream > 126 MB L2; tape holds GBs)"}


class ClockSampler:
    """nvidia-smi-equivalent clock/throttle sampling (NVML) during the timed region."""
    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
             0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.stop_ev = [], 0, threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            self.stop_ev.wait(0.1)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "samples": len(self.samples),
                "reasons": [n for b, n in self.NAMES.items() if self.reasons & b and b != 0x1]}


def algorithmic_bytes(dim: int, N: int, A: float) -> dict:
    """Per-launch algorithmic bytes of each kernel class:
    the minimum HBM traffic of the kernel's own inputs/outputs, N particles and
    A active grid nodes per launch (fp32; record s = 4(2d + 2d^2) bytes)."""
    s = 4 * (2 * dim + 2 * dim * dim)
    dd, d = 4 * dim * dim, 4 * dim
    node = 16  # (P, M) or (U, z) float4 per node
    return {
        "p2g": N * (s + 4 + dd) + A * node,                      # S_t, aid -> F_{t+1}; grid flush
        "grid_op": A * 2 * node,                                  # (P, M) -> (U, z)
        "g2p": N * (d + d + d + dd) + A * node,                   # x_t -> x, v, C; read U
        "g2p_grad": N * (d + 2 * d + dd) + A * node,              # x_t, (xb, vb, Cb)' -> U_bar tiles
        "g2p_grad_gather": N * (d + 2 * d + dd + d) + A * node,   # x_t, (xb, vb, Cb)', U -> xb_t partial
        "canon": N * 17,                                          # sigma, pid, cell -> sigma, pid
        "grid_op_grad": A * 4 * node,                             # P,M, U, Ub -> (Pb, Mb)
        "p2g_grad": N * (s + 4 + dd + d + s) + A * node,          # S_t, aid, Fb', xb -> S_bar_t
    }


# The paper's one timing of this path: Table 1, DiffTaichi diffmpm,
# 2D, 6.4K particles, 0.11 ms forward + 0.15 ms backward per time step on a GTX 1080 Ti
# -> 6,400 / 0.26 ms = 24.6 M particle-steps/s.  Only the 2D 6.4K-particle
# workload (c2) matches it; every other config reports null.
PAPER_TABLE1_2D_6K4 = 6400 / 0.26e-3


def _vs_baseline(p: dict, value: float):
    if p.get("name") == "c2" and p["dim"] == 2:
        return value / PAPER_TABLE1_2D_6K4
    return None


def _traffic(kernel: str):
    """dram bytes per launch from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# -------------------------------------------------------------- CPU oracle
def host_info():
    """the host the CPU baseline ran on: logical cores and the lscpu model name"""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def oracle_sample(p, inp, steps=1, precision="f64"):
    """time the CPU oracle (as it stands) on a bounded sample: all particles of the
    episode, `steps` time steps of forward + loss + backward, one thread (fp64 build, or the
    fp32 build of the same C source)."""
    from oracle import Oracle
    o = Oracle(p, precision)
    if inp.get("mat") is not None and np.any(inp["mat"]):
        o.set_materials(inp["mat"])
    t0 = time.perf_counter()
    o.run(inp["x"], inp["v"], inp["C"], inp["F"], inp["aid"], inp["theta"], steps=steps,
          k_ckpt=steps)
    dt = time.perf_counter() - t0
    return len(inp["x"]) * steps / dt, dt


def run_reference(args):
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    from paper_1910_00935_b200 import workloads as W
    p, _, scaling = _workload(args.config, 1)
    inp = W.make_inputs(p)
    steps = 1
    for _ in range(args.warmup):
        oracle_sample(p, inp, steps)
    times = []
    for _ in range(args.steps):
        _, dt = oracle_sample(p, inp, steps)
        times.append(dt)
    N = len(inp["x"])
    total = sum(times)
    value = N * steps * args.steps / total
    sample = (f"{p['name']} rank-0 episode, all {N:,} particles, {steps} time step(s) of "
              f"forward + loss + backward per bench step (fp64 oracle)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _describe(p, N, 1, 1, p["k_ckpt"]),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": sample, "host": host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _pick_k(p, N, per, T, dev, use_dist=False):
    """Smallest checkpoint interval whose tape fits in 90% of free HBM (Appendix D.2:
    k trades re-forward work for memory; on a 180 GB B200 the 1M-particle cube fits k = 2).
    Under torchrun every rank must run the same k (the same re-forward work): the ranks agree
    on the MIN of their free memory, and the largest shard sizes the workspace."""
    import torch
    from paper_1910_00935_b200 import mpm
    free, _ = torch.cuda.mem_get_info(dev)
    if use_dist:
        import torch.distributed as dist
        t = torch.tensor([float(free), -float(per)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        free, per = int(t[0].item()), int(-t[1].item())
    for k in (1, 2, 4, 8, 16, 32, 64, 128):
        if k > T:
            break
        probe = mpm.sim_from_config(p, N, episodes=per, max_steps=T, k_ckpt=k, probe_only=True)
        need = probe.workspace_bytes
        probe.close()
        if need < 0.9 * free:
            return k
    return int(p.get("k_ckpt", 32))


# -------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1910_00935_b200 import mpm, workloads as W

    rank, world, local = _env_int("RANK", 0), _env_int("WORLD_SIZE", 1), _env_int("LOCAL_RANK", 0)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # under torchrun the process group is set up even at world size 1 (the NCCL path runs as
    # it would on N GPUs: init, the agreed k, the gradient all-reduce, max-over-ranks timing)
    use_dist = world > 1 or "TORCHELASTIC_RUN_ID" in os.environ
    if use_dist:
        # NCCL over NVLink/NVSwitch; BENCH_DIST_BACKEND=gloo only for exercising the
        # multi-rank code path with several ranks on one GPU (NCCL rejects that)
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    from paper_1910_00935_b200.dist import allreduce_shared_grad, max_over_ranks
    if args.shard_of and world > 1:
        raise SystemExit("--shard-of is a one-process projection; run it without torchrun")
    p, shard, scaling = _workload(args.config, args.shard_of or world, rank)
    per = len(shard)
    T = int(p["steps"])
    if args.config == "c4":
        inps = [W.make_inputs(p, episode=e) for e in shard]
    else:
        inps = [W.make_inputs(p, rank=rank)]
    N = len(inps[0]["x"])
    cat = lambda key: np.ascontiguousarray(np.stack([i[key] for i in inps]))  # noqa: E731
    host = {key: torch.from_numpy(cat(key)).pin_memory() for key in ("x", "v", "C", "F", "aid")}
    host["theta"] = torch.from_numpy(inps[0]["theta"]).pin_memory()
    devin = {key: t.to(dev) for key, t in host.items()}

    k = int(args.k_ckpt) if args.k_ckpt else _pick_k(p, N, per, T, dev, use_dist)
    sim = mpm.sim_from_config(p, N, episodes=per, max_steps=T, k_ckpt=k)
    if any(np.any(i["mat"]) for i in inps):  # fluid particles (R23): a property of the workload
        sim.set_materials(cat("mat"))
    nth = sim.n_theta
    shared_len = nth if nth > 0 else per * p["dim"]
    loss_d = torch.zeros(per, device=dev)
    shared_d = torch.zeros(shared_len, device=dev)
    gdev = {"dx0": torch.empty((per, N, p["dim"]), device=dev),
            "dv0": torch.empty((per, N, p["dim"]), device=dev),
            "dC0": torch.empty((per, N, p["dim"], p["dim"]), device=dev),
            "dF0": torch.empty((per, N, p["dim"], p["dim"]), device=dev),
            "dtheta": torch.empty(max(nth, 1), device=dev)}
    loss_h = torch.zeros(per).pin_memory()
    shared_h = torch.zeros(shared_len).pin_memory()

    def step(src, loss_buf, shared_buf, grads_out):
        sim.set_state(src["x"], src["v"], src["C"], src["F"], src["aid"])
        sim.set_controller(src["theta"])
        sim.forward(T)
        sim.loss(loss_buf)
        sim.backward(T)
        if nth > 0:
            sim.grads({"dtheta": shared_buf, **(grads_out or {})})
        else:
            if grads_out:
                sim.grads(grads_out)
            sim.grad_v0_sum(shared_buf)
        if use_dist:
            # the one exchange of the path: sum of the shared-parameter gradient over ranks
            if shared_buf.is_cuda:
                allreduce_shared_grad(shared_buf)
            else:
                t = shared_buf.to(dev)
                allreduce_shared_grad(t)
                shared_buf.copy_(t)

    def timed(K, fn):
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(K):
            fn()
        e.record()
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier()
        return max_over_ranks(s.elapsed_time(e), dev)

    dev_step = lambda: step(devin, loss_d, shared_d, gdev)  # noqa: E731
    host_step = lambda: step(host, loss_h, shared_h, None)  # noqa: E731

    for _ in range(args.warmup):
        dev_step()
    # active grid nodes (A) for the algorithmic byte count: the grid store keeps every recorded
    # step's node tiles, so A is averaged over 9 steps spread over the horizon
    sim.set_state(devin["x"], devin["v"], devin["C"], devin["F"], devin["aid"])
    sim.set_controller(devin["theta"])
    sim.forward(T)
    a_steps = sorted({min(T - 1, (T - 1) * j // 8) for j in range(9)})
    A = float(np.mean([sim.active_nodes(t) for t in a_steps])) / per

    # timed region (CUDA graphs replayed; no per-kernel events so nothing perturbs it)
    l0 = sim.launch_count()
    clocks = ClockSampler(local)
    with clocks:
        ms = timed(args.steps, dev_step)
    launches = sim.launch_count() - l0
    # per-kernel device time: a second timed region with CUDA events bracketing every
    # library launch on the library's stream (eager launches; graphs are off while profiling)
    sim.reset_kernel_stats()
    sim.set_profiling(True)
    ms_prof = timed(args.steps, dev_step)
    stats = sim.kernel_stats()
    sim.set_profiling(False)
    ms_e2e = timed(args.steps, host_step)

    # units of all ranks (C4 shards may differ by one episode: count them exactly)
    if use_dist:
        tot = torch.tensor([float(N) * per * T * args.steps], dtype=torch.float64, device=dev)
        dist.all_reduce(tot)
        particle_steps = float(tot.item())
    else:
        particle_steps = float(N) * per * T * args.steps
    value = particle_steps / (ms / 1e3)
    e2e_value = particle_steps / (ms_e2e / 1e3)
    h2d = sum(int(t.numel() * t.element_size()) for t in host.values())
    d2h = int(loss_h.numel() * 4 + shared_h.numel() * 4)

    # roofline of the dominant kernel (largest share of device time)
    peak, peak_src = _peaks()
    alg = algorithmic_bytes(p["dim"], N * per, A * per)
    if not stats.get("canon", (0, 0))[1]:  # small problems: p2g orders its blocks itself (no canon pass)
        alg["p2g"] += alg["canon"]
    kern = {kname: v for kname, v in stats.items() if kname in alg and v[1] > 0}
    dom = max(kern, key=lambda kk: kern[kk][0])
    dom_ms, dom_n = kern[dom]
    total_ms = sum(v[0] for v in stats.values())
    achieved = alg[dom] / (dom_ms / dom_n / 1e3) / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": _traffic(dom), "peak_source": peak_src,
                "alg_bytes_per_launch": alg[dom], "avg_launch_us": 1e3 * dom_ms / dom_n,
                "share_of_kernel_time": dom_ms / total_ms if total_ms else None,
                "active_nodes_per_episode": A,
                "kernel_ms": {kk: round(v[0] / args.steps, 3) for kk, v in stats.items() if v[1]},
                # every particle / node kernel's algorithmic GB/s over the peak (the dominant one is `frac`)
                "kernel_frac": {kk: round(alg[kk] / (v[0] / v[1] / 1e3) / 1e9 / peak, 4) for kk, v in kern.items()},
                "profiled_ms_per_step": ms_prof / args.steps,
                "kernel_launches_per_step": {kk: v[1] // args.steps for kk, v in stats.items() if v[1]}}
    # whole-step effective bandwidth against the SURVEY 8(d) byte model
    s_rec = 4 * (2 * p["dim"] + 2 * p["dim"] ** 2)
    B_p = (2 * s_rec + 4) * (1 + (k - 1) / k) + (3 * s_rec + 12 * p["dim"] + 4)
    B_g = 8 * (p["dim"] + 1) * (1 + (k - 1) / k) + 8 * (p["dim"] + 1) + 8 * p["dim"]
    step_bytes = (N * B_p + A * B_g) * per * T
    roofline["step_model_bytes"] = step_bytes
    roofline["step_effective_GBps_per_gpu"] = step_bytes / (ms / args.steps / 1e3) / 1e9
    roofline["step_frac"] = roofline["step_effective_GBps_per_gpu"] / peak

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v_cpu, dt_cpu = oracle_sample(p, inps[0], steps=4)
        v_f32, dt_f32 = oracle_sample(p, inps[0], steps=4, precision="f32")
        cpu = {"value": v_cpu, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{p['name']} episode 0, all {N:,} particles, 4 time steps of forward + "
                         f"loss + backward, fp64, single thread ({dt_cpu:.1f} s)",
               "f32_build": {"value": v_f32, "unit": UNIT, "seconds": dt_f32},
               "host": host_info()}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": scaling, "vs_baseline": _vs_baseline(p, value), "dtype": "f32", "data": "synthetic",
                "config": _describe(p, N, per, world, k), "roofline": roofline,
                "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e / args.steps,
                        "outputs": "per step: the initial state S_0 (x, v, C, F, actuator ids) + theta copied "
                                   "in from pinned host memory; the loss and the shared-parameter gradient "
                                   "(theta_bar, or sum_p dL/dv0_p for the cube) read back; the device-timed "
                                   "`value` additionally writes the per-particle gradients dL/d(x0, v0, C0, F0) "
                                   "into device buffers"},
                "gpu_launches": int(launches), "clocks": clocks.summary(),
                "loss": [float(x) for x in loss_d.cpu()]}
        if args.shard_of:
            line["shard_of"] = {"n_gpus": args.shard_of, "rank": 0, "episodes": per,
                                "note": "one GPU running rank 0's share of an N-GPU job (no all-reduce): "
                                        "`value` is this GPU's own rate, not a whole-job number"}
        print(json.dumps(line), flush=True)
    sim.close()
    if use_dist:
        dist.destroy_process_group()
    return 0


def run_dd(args):
    """ONE body decomposed into `--dd` slab subdomains (include/mpm.h mpm_dd_*), one
    process driving one handle per slab -- on as many GPUs as are visible (round robin), else all on
    cuda:0.  Same metric (fwd+bwd particle-steps/s of the whole body); k = 1 (the decomposed
    tape keeps every state), so the horizon is capped by memory: BENCH_HORIZON (default 256)."""
    import torch
    from paper_1910_00935_b200 import mpm, workloads as W
    p = W.config(args.config, steps=int(os.environ.get("BENCH_HORIZON", 256)))
    if int(p.get("n_act", 0)) != 0:
        raise SystemExit("--dd needs a passive body (c1a, c1b, c5)")
    T, G = int(p["steps"]), int(args.dd)
    inp = W.make_inputs(p)
    N = len(inp["x"])
    B = 4 if p["dim"] == 3 else 8
    nb = -(-p["n_grid"] // B)
    xs = inp["x"][:, 0].astype(np.float32)
    bx = np.floor(xs * np.float32(p["n_grid"]) - np.float32(0.5)).astype(np.int64) // B
    # slabs with about equal particle counts (block-column boundaries)
    cuts = sorted({min(nb - 1, max(1, int(np.quantile(bx, g / G)))) for g in range(1, G)})
    bounds = [0] + cuts + [nb]
    ndev = max(1, torch.cuda.device_count())
    sims, sel, streams = [], [], []
    for g, (lo, hi) in enumerate(zip(bounds[:-1], bounds[1:])):
        ids = np.nonzero((bx >= lo) & (bx < hi))[0].astype(np.int32)
        dev = g % ndev
        torch.cuda.set_device(dev)
        st = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(st):
            # capacity: the slab's particles plus room for the body drifting across slabs
            cap = min(N, int(len(ids) + max(0.5 * len(ids), N / G))) + 8192
            sims.append(mpm.sim_from_config(p, cap, max_steps=T, k_ckpt=1, subdomain=(lo, hi, N)))
        sel.append(ids)
        streams.append(st)
    mpm.dd_link(sims)
    dev_in = []
    for sim, ids, g in zip(sims, sel, range(len(sims))):
        d = g % ndev
        dev_in.append({k: torch.from_numpy(np.ascontiguousarray(inp[k][ids])).to(f"cuda:{d}") for k in "xvCF"} |
                      {"ids": torch.from_numpy(ids).to(f"cuda:{d}")})
    for d in range(ndev):  # the inputs were copied on torch's current stream, the handles use their own
        torch.cuda.synchronize(d)

    def step():
        for sim, di in zip(sims, dev_in):
            sim.set_state_ids(di["x"], di["v"], di["C"], di["F"], di["ids"])
        mpm.dd_forward(sims, T)
        mpm.dd_loss(sims)
        mpm.dd_backward(sims, T)

    for _ in range(args.warmup):
        step()
    for d in range(ndev):
        torch.cuda.synchronize(d)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ndev)]
    for d in range(ndev):
        with torch.cuda.device(d):
            ev[d][0].record(streams[d])
    for _ in range(args.steps):
        step()
    for d in range(ndev):
        with torch.cuda.device(d):
            ev[d][1].record(streams[d])
    for d in range(ndev):
        torch.cuda.synchronize(d)
    ms = max(ev[d][0].elapsed_time(ev[d][1]) for d in range(min(ndev, len(sims))))
    value = float(N) * T * args.steps / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": min(ndev, G), "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{p['name']}: one body of {N:,} particles over {G} slab subdomains (f3) on "
                                   f"{min(ndev, G)} GPU(s), {p['n_grid']}^{p['dim']} grid, {T} steps, k = 1",
                       "slabs_block_x": bounds, "particles_per_slab": [int(len(s)) for s in sel]},
            "gpu_launches": int(sum(s.launch_count() for s in sims))}
    print(json.dumps(line), flush=True)
    for s in sims:
        s.close()
    return 0


def run_ours_on_stream(args):
    """the library captures its forward/backward tapes as CUDA graphs, which needs a
    non-default stream: run the whole arm on a dedicated torch stream."""
    import torch
    local = _env_int("LOCAL_RANK", 0) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    with torch.cuda.stream(torch.cuda.Stream()):
        return run_ours(args)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=["c1a", "c1b", "c2", "c2cl", "c3", "c3cl", "c3liquid", "c4", "c5"])
    ap.add_argument("--k-ckpt", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dd", type=int, default=0, help="f3: one body over this many slab subdomains (one process)")
    ap.add_argument("--shard-of", type=int, default=0,
                    help="one GPU runs rank 0's share of an N-GPU job (C4: 64/N episodes): the per-rank "
                         "compute of the N-GPU run without its all-reduce, a strong-scaling projection")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.dd:
        return run_dd(args)
    return run_ours_on_stream(args)


if __name__ == "__main__":
    sys.exit(main())
