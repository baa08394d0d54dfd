#!/usr/bin/env python
"""Benchmark of the B200 free-space Spectral Ewald hot path (fse::total_sum).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2] [--no-cpu-baseline]

A step = one fse::total_sum (spread -> FFT -> k-space scale -> IFFT ->
quadrature, plus the real-space pair sum and the self term) over the whole
synthetic workload.  Default workload: BASELINE.json configs[1] ("cfg2"):
stokeslet, N = NT = 1e6 uniform in [0,1)^3, N(0,1) forces, xi=110, rc=0.045,
M=288, P=24 (Mtilde=312, FFT grid D=624).

value : targets/s, inputs resident in HBM, CUDA events on the context stream
        over exactly K steps (fse_cuda_total_sum_dev), max over ranks;
e2e   : targets/s through the reference-facing C-ABI call with HOST buffers
        (fse_cuda_total_sum, pinned inputs): H2D of positions+forces and D2H
        of the velocities inside the timed region, wall clock;
roofline : the dominant kernel of the step, achieved = algorithmic bytes or
        flops per launch / its CUDA-event duration;
cpu_baseline : the reference compiled from its own sources (oracle/_ref) timed
        on this host at the SAME workload: one full fse::total_sum call (its
        Green's precompute excluded, as harness.hpp:50 does), rank 0, N=1 only;
--impl reference : the same reference call, warm-up + timed steps until K or a
        time budget (--ref-budget-s) is reached (reported as "steps"); inputs
        from the reference-side generator (oracle/ref_capi.cpp), so the arm
        never loads the product library.

N > 1 (torchrun, or `--gpus N` which relaunches itself under torchrun): one
evaluation decomposed into N z-slabs (slabs.py);
--replicas runs N independent full evaluations instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs (kind, generator, N, xi, rc, M, P, distinct targets)
WORKLOADS = {
    "cfg1": dict(kind=0, wl=1, n=10_000, xi=28.0, rc=0.15, M=80, P=16, tol=1e-8,
                 desc="stokeslet N=1e4 uniform [0,1)^3, xi=28 rc=0.15 M=80 P=16"),
    "cfg2": dict(kind=0, wl=1, n=1_000_000, xi=110.0, rc=0.045, M=288, P=24, tol=1e-10,
                 desc="stokeslet N=1e6 uniform [0,1)^3, xi=110 rc=0.045 M=288 P=24"),
    "cfg3": dict(kind=1, wl=3, n=100_000, xi=40.0, rc=0.12, M=128, P=20, tol=1e-8,
                 desc="stresslet N=1e5 on the sphere r=0.5, xi=40 rc=0.12 M=128 P=20"),
    "cfg4": dict(kind=2, wl=4, n=1_000_000, xi=110.0, rc=0.045, M=288, P=24, tol=1e-10,
                 desc="rotlet N=1e6 in 32 Gaussian blobs sigma=0.03, xi=110 rc=0.045 M=288 P=24"),
    "cfg5": dict(kind=0, wl=5, n=8_000_000, xi=220.0, rc=0.022, M=576, P=24, tol=1e-10,
                 desc="stokeslet N=8e6 + 8e6 distinct targets uniform, xi=220 rc=0.022 M=576 P=24"),
    # tolerance-consistent variants: (rc, M, P) from the reference's
    # select_parameters at the same xi and tolerance (estimates.cpp:81-126)
    "cfg1t": dict(kind=0, wl=1, n=10_000, xi=28.0, tol=1e-8, select=True,
                  desc="cfg1 inputs, (rc, M, P) = select_parameters(xi=28, tol=1e-8)"),
    "cfg2t": dict(kind=0, wl=1, n=1_000_000, xi=110.0, tol=1e-10, select=True,
                  desc="cfg2 inputs, (rc, M, P) = select_parameters(xi=110, tol=1e-10)"),
    "cfg3t": dict(kind=1, wl=3, n=100_000, xi=40.0, tol=1e-8, select=True,
                  desc="cfg3 inputs, (rc, M, P) = select_parameters(xi=40, tol=1e-8)"),
    "cfg4t": dict(kind=2, wl=4, n=1_000_000, xi=110.0, tol=1e-10, select=True,
                  desc="cfg4 inputs, (rc, M, P) = select_parameters(xi=110, tol=1e-10)"),
    # M = 834, D = 1730 = 2 x 5 x 173: generic Stockham stage of radix 173 at one
    # CTA per SM (227 KB of shared memory), ~135 GB of HBM, ~2.7 s per call
    "cfg5t": dict(kind=0, wl=5, n=8_000_000, xi=220.0, tol=1e-10, select=True,
                  desc="cfg5 inputs, (rc, M, P) = select_parameters(xi=220, tol=1e-10)"),
}


def quadratic_sum(strengths) -> float:
    """strength_quadratic_sum (kernels.cpp:105-110): sequential sum of c_i^2."""
    return float(np.cumsum((strengths * strengths).ravel())[-1])


def workload_config(w, strengths, lib):
    """The workload's EwaldConfig: explicit (rc, M, P), or the tolerance-consistent
    choice of select_parameters (lib = the product package or oracle.refimpl)."""
    if not w.get("select"):
        return lib.make_config(1.0, w["xi"], w["rc"], w["M"], w["P"])
    cfg, feasible = lib.select_parameters(w["kind"], w["n"], 1.0, quadratic_sum(strengths),
                                          w["xi"], w["tol"])
    if not feasible:
        raise SystemExit(f"select_parameters: tolerance {w['tol']} infeasible")
    return cfg
KIND_NAMES = ["stokeslet", "stresslet", "rotlet"]
SEED = 20260101


def metric_name(w):
    return (f"{KIND_NAMES[w['kind']]} targets/sec at N={w['n']:.0e}, fp64 tol {w['tol']:.0e}, "
            "1/2/4/8 B200; % of roofline")


# ------------------------------------------------------------------ output
# The JSON line is the only thing on stdout: file descriptor 1 is pointed at
# stderr for the rest of the run (NCCL's version banner, library prints), and
# the line goes to a saved copy of the original stdout.
_JSON_OUT = None


def emit(line: dict):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def _stdout_to_stderr():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


# ------------------------------------------------------------------ dist
class Dist:
    def __init__(self, force_group=False):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.grouped = self.world > 1 or force_group
        if self.grouped:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", str(self.rank))
            os.environ.setdefault("WORLD_SIZE", str(self.world))
            import torch
            import torch.distributed as td
            self.torch, self.td = torch, td
            backend = "nccl" if torch.cuda.is_available() else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(self.local)
            td.init_process_group(backend=backend)
            self.dev = torch.device("cuda", self.local) if backend == "nccl" else torch.device("cpu")

    def barrier(self):
        if self.grouped:
            self.td.barrier()

    def max(self, v: float) -> float:
        if not self.grouped:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.dev)
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.grouped:
            self.td.destroy_process_group()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampled during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, flag in zip(names, parts[3:7]):
                if flag.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ roofline
def peaks():
    p = {"hbm_gbs": 6650.0, "hbm_src": "fallback (B200_PROFILING.md)"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        if m.get("hbm_gbs"):
            p = {"hbm_gbs": float(m["hbm_gbs"]), "hbm_src": "measured (MEASURED_PEAKS.json)"}
    return p


# FP64 flops of one accepted real-space pair, calibrated from ncu's SASS
# instruction counts of k_realspace (2 DFMA + DMUL + DADD thread instructions per
# accepted pair; tools/pair_flops.py, profiles/r02/realspace_pair_flops.txt):
# stokeslet cfg2 101.8, stresslet cfg3 163.0, rotlet cfg4 96.8
PAIR_FLOPS = {0: 102.0, 1: 163.0, 2: 97.0}


def stage_models(w, cfg, n, nt, rs_pairs=None):
    """Algorithmic work per launch: flops or bytes."""
    a = 9 if w["kind"] == 1 else 3
    P, D = cfg.P, cfg.D
    Mt = cfg.Mtilde
    Dh = D // 2 + 1
    R = 8.0 * Mt ** 3            # compact real grid, one component
    B = 16.0 * Mt * Mt * Dh      # after the z pass
    Cs = 16.0 * Mt * D * Dh      # after the y pass
    G = 8.0 * D * D * Dh         # real half-spectrum multiplier
    models = {
        # FP64 FMA-bound: 2 a P^3 flops per source, 2*3 P^3 per target
        "spread": ("fp64", 2.0 * a * P ** 3 * n),
        "gather": ("fp64", 2.0 * 3 * P ** 3 * nt),
        # HBM-bound pruned passes, each reading its input and writing its output once:
        # z (R -> B), y (B -> C); fused x-pass + multiplier (C, G -> C); inverse y, z
        "fft_forward": ("hbm", a * (R + B) + a * (B + Cs)),
        "kscale": ("hbm", a * Cs + G + 3 * Cs),
        "fft_inverse": ("hbm", 3 * (Cs + B) + 3 * (B + R)),
    }
    if rs_pairs:
        models["realspace"] = ("fp64", PAIR_FLOPS[w["kind"]] * rs_pairs)
    return models


# ------------------------------------------------------------------ ours, partitioned
def run_dist(args, dist: Dist):
    """N > 1: one evaluation of the workload with the particles PARTITIONED over N
    x-slabs (fse_cuda_dist_*): each rank holds only
    the points it owns (fse_dist_owner) and the library exchanges ghost sources and
    targets, the two spectrum transposes and the ghost partial sums over NCCL
    (grouped ncclSend / ncclRecv).  Total work fixed as N grows: strong scaling."""
    import torch
    import paper_1607_04808_b200 as fse

    w = WORKLOADS[args.workload]
    ctx = fse.Context(dist.local)
    system, tgt = fse.generate_workload(w["wl"], w["n"], SEED)  # same stream on every rank
    tas = tgt is None
    targets = system.positions if tas else tgt
    n_total, nt_total = system.size(), targets.shape[0]
    cfg = workload_config(w, system.strengths, fse)
    G, r = dist.world, dist.rank
    own_s = np.nonzero(fse.dist_owner(cfg, G, system.positions) == r)[0]
    own_t = own_s if tas else np.nonzero(fse.dist_owner(cfg, G, targets) == r)[0]
    hp = ctx.host_alloc((own_s.size, 3))
    hs = ctx.host_alloc((own_s.size, system.strengths.shape[1]))
    hp[...] = system.positions[own_s]
    hs[...] = system.strengths[own_s]
    ht = hp if tas else ctx.host_alloc((own_t.size, 3))
    if not tas:
        ht[...] = targets[own_t]
    hu = ctx.host_alloc((own_t.size, 3))
    del system, tgt, targets
    n_own, nt_own = own_s.size, own_t.size
    d_pos = ctx.dev_alloc(max(hp.nbytes, 8))
    d_str = ctx.dev_alloc(max(hs.nbytes, 8))
    d_tgt = d_pos if tas else ctx.dev_alloc(max(ht.nbytes, 8))
    d_u = ctx.dev_alloc(max(24 * nt_own, 8))

    def upload():
        if hp.nbytes:
            ctx.memcpy(d_pos, hp.ctypes.data, hp.nbytes)
            ctx.memcpy(d_str, hs.ctypes.data, hs.nbytes)
        if not tas and ht.nbytes:
            ctx.memcpy(d_tgt, ht.ctypes.data, ht.nbytes)

    upload()
    green = ctx.precompute_mollified_green(int(fse.green_kind_for(w["kind"])), cfg.Ltilde,
                                           cfg.Mtilde, cfg.sf)
    # NCCL communicator of the library: rank 0's unique id, broadcast over the
    # torch.distributed group
    uid = torch.zeros(128, dtype=torch.uint8, device=dist.dev)
    if r == 0:
        uid[:] = torch.frombuffer(bytearray(fse.nccl_unique_id()), dtype=torch.uint8)
    dist.td.broadcast(uid, 0)
    handle = ctx.dist_create(r, G, bytes(uid.cpu().numpy().tobytes()))

    def step():
        ctx.dist_total_sum(handle, cfg, w["kind"], d_pos, d_str, n_own, n_total, d_tgt, nt_own,
                           tas, green, d_u)

    for _ in range(args.warmup):
        step()
    clocks = ClockSampler(dist.local)
    clocks.start()
    time.sleep(0.3)
    launches0 = ctx.launch_count
    dist.barrier()
    torch.cuda.synchronize()
    ctx.mark()
    for _ in range(args.steps):
        step()
    ctx.mark()
    dev_ms = ctx.elapsed_ms()
    launches = ctx.launch_count - launches0
    clk = clocks.stop()
    dist.barrier()
    max_ms = dist.max(dev_ms)

    # e2e: each rank's owned inputs from pinned host memory, its owned velocities back
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(max(1, args.steps)):
        upload()
        step()
        if hu.nbytes:
            ctx.memcpy(hu.ctypes.data, d_u, hu.nbytes)
    e2e_s = dist.max(time.perf_counter() - t0)
    h2d = hp.nbytes + hs.nbytes + (0 if tas else ht.nbytes)

    a = 9 if w["kind"] == 1 else 3
    flops = 2.0 * a * cfg.P ** 3 * n_total + 2.0 * 3 * cfg.P ** 3 * nt_total
    fp64_peak = args.fp64_peak or ctx.measure_fp64_peak()
    ach = flops / G / (max_ms / args.steps * 1e-3) / 1e12
    value = nt_total * args.steps / (max_ms * 1e-3)
    counts = torch.tensor([n_own, nt_own], dtype=torch.float64, device=dist.dev)
    allc = [torch.zeros_like(counts) for _ in range(G)]
    dist.td.all_gather(allc, counts)
    line = {
        "metric": metric_name(w), "value": value, "unit": "targets/s", "n_gpus": G,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: SURVEY 8(d) generator {w['wl']} (mt19937_64 seed {SEED}), each "
                "rank keeps the points its slab owns, no dataset",
        "config": {"workload": f"{args.workload}: {w['desc']}", "kind": KIND_NAMES[w["kind"]],
                   "N": n_total, "NT": nt_total, "Mtilde": cfg.Mtilde, "fft_grid": cfg.D,
                   "parallelism": f"x-slabs x{G}: partitioned particles, NCCL ghost / "
                                  "transpose / partial-sum exchanges (fse_cuda_dist_total_sum)",
                   "owned_per_rank": [[int(c[0].item()), int(c[1].item())] for c in allc],
                   "l2": working_set_note(w, cfg)},
        "e2e": {"value": nt_total * max(1, args.steps) / e2e_s, "unit": "targets/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(hu.nbytes),
                "api": "fse_cuda_dist_total_sum (owned points from pinned host memory per rank)"},
        "roofline": {"bound": "fp64", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s",
                     "frac": ach / fp64_peak, "kernel": "step (spread + quadrature work / rank)",
                     "traffic": None},
        "gpu_launches": int(launches),
        "clocks": clk,
        "cpu_baseline": None,
    }
    if r == 0:
        emit(line)
    for p in (d_pos, d_str, d_u) + (() if tas else (d_tgt,)):
        ctx.dev_free(p)


# ------------------------------------------------------------------ ours
def run_ours(args, dist: Dist):
    import paper_1607_04808_b200 as fse

    w = WORKLOADS[args.workload]
    ctx = fse.Context(dist.local)
    system, tgt = fse.generate_workload(w["wl"], w["n"], SEED + dist.rank)
    targets = system.positions if tgt is None else tgt
    n, nt = system.size(), targets.shape[0]
    tas = 1 if tgt is None else 0
    cfg = workload_config(w, system.strengths, fse)
    t0 = time.perf_counter()
    green = ctx.precompute_mollified_green(int(fse.green_kind_for(w["kind"])), cfg.Ltilde,
                                           cfg.Mtilde, cfg.sf)
    precompute_s = time.perf_counter() - t0

    # inputs resident in HBM
    a = system.strengths.shape[1]
    d_pos = ctx.dev_alloc(system.positions.nbytes)
    d_str = ctx.dev_alloc(system.strengths.nbytes)
    d_tgt = d_pos if tas else ctx.dev_alloc(targets.nbytes)
    d_u = ctx.dev_alloc(8 * 3 * nt)
    ctx.memcpy(d_pos, system.positions.ctypes.data, system.positions.nbytes)
    ctx.memcpy(d_str, system.strengths.ctypes.data, system.strengths.nbytes)
    if not tas:
        ctx.memcpy(d_tgt, targets.ctypes.data, targets.nbytes)

    def step(tm=None):
        ctx.total_sum_dev(cfg, w["kind"], d_pos, d_str, n, 1.0, d_tgt, nt, green, d_u,
                          targets_are_sources=tas, timings=tm)

    for _ in range(args.warmup):
        step()
    dist.barrier()
    clocks = ClockSampler(dist.local)
    clocks.start()
    time.sleep(0.3)
    launches0 = ctx.launch_count
    kms = np.zeros(11)
    tm = fse.StageTimings()
    ctx.mark()
    for _ in range(args.steps):
        step(tm)
        kms += np.array(ctx.kernel_ms())
    ctx.mark()
    dev_ms = ctx.elapsed_ms()
    launches = ctx.launch_count - launches0
    clk = clocks.stop()
    dist.barrier()
    max_ms = dist.max(dev_ms)
    # stage breakdown from extra untimed steps with the real-space stream
    # serialised (the overlapped events in the timed steps interleave)
    ctx.set_overlap(False)
    kms[:] = 0
    nbrk = 2
    tm = fse.StageTimings()
    for _ in range(nbrk):
        step(tm)
        kms += np.array(ctx.kernel_ms())
    ctx.set_overlap(True)
    kms /= nbrk

    # e2e through the host-buffer C-ABI call, pinned inputs
    hp = ctx.host_alloc(system.positions.shape)
    hs = ctx.host_alloc(system.strengths.shape)
    hp[...] = system.positions
    hs[...] = system.strengths
    hsys = fse.SourceSystem(hp, hs, 1.0)
    ht = hp if tas else ctx.host_alloc(targets.shape)
    if not tas:
        ht[...] = targets
    hu = ctx.host_alloc((targets.shape[0], 3))  # pinned result buffer
    ctx.total_sum(hsys, w["kind"], cfg, ht, green, targets_are_sources=tas, out=hu)  # warm
    dist.barrier()
    e2e_steps = max(1, args.steps)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        u_host = ctx.total_sum(hsys, w["kind"], cfg, ht, green, targets_are_sources=tas, out=hu)
    e2e_s = dist.max(time.perf_counter() - t0)
    h2d = hp.nbytes + hs.nbytes + (0 if tas else ht.nbytes)
    d2h = u_host.nbytes

    # roofline of the dominant kernel
    names = ["spread", "fft_forward", "kscale", "fft_inverse", "gather", "realspace"]
    stage_ms = {"source_prep": kms[0], "spectrum_memset": kms[1], "spread": kms[2],
                "fft_forward": kms[3], "kscale": kms[4], "fft_inverse": kms[5],
                "target_prep": kms[6], "gather": kms[7], "realspace_binning": kms[8],
                "realspace": kms[9], "call": kms[10]}
    rs_cand, rs_pairs = ctx.realspace_counts()
    models = stage_models(w, cfg, n, nt, rs_pairs)
    pk = peaks()
    fp64_peak = args.fp64_peak
    if fp64_peak is None:
        fp64_peak = ctx.measure_fp64_peak()
    stage_roof = {}
    for nm in names:
        if nm not in models or stage_ms[nm] <= 0:
            continue
        bound, work = models[nm]
        if bound == "hbm":
            ach = work / (stage_ms[nm] * 1e-3) / 1e9
            stage_roof[nm] = {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"],
                              "unit": "GB/s", "frac": ach / pk["hbm_gbs"]}
        else:
            ach = work / (stage_ms[nm] * 1e-3) / 1e12
            stage_roof[nm] = {"bound": "fp64", "achieved": ach, "peak": fp64_peak,
                              "unit": "TFLOP/s", "frac": ach / fp64_peak}
    dom = max((nm for nm in names if stage_ms.get(nm, 0) > 0 and nm in stage_roof),
              key=lambda k: stage_ms[k])
    roof = dict(stage_roof[dom])
    roof["kernel"] = dom
    roof["ms"] = stage_ms[dom]
    roof["peak_src"] = pk["hbm_src"] if roof["bound"] == "hbm" else \
        "measured in this run (DFMA loop, fse_cuda_fp64_peak)"
    roof["traffic"] = traffic_for(args.workload, dom)

    cpu = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_line(w)

    value = dist.world * nt * args.steps / (max_ms * 1e-3)
    line = {
        "metric": metric_name(w), "value": value, "unit": "targets/s", "n_gpus": dist.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
        # N = 1 is the base of the strong-scaling series of run_dist (one evaluation
        # split over N GPUs); --replicas at N > 1 is weak scaling (N evaluations)
        "higher_is_better": True, "scaling": "weak" if dist.world > 1 else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: SURVEY 8(d) generator {w['wl']} (mt19937_64 seed {SEED}+rank), "
                "no dataset",
        "config": {"workload": f"{args.workload}: {w['desc']}", "kind": KIND_NAMES[w["kind"]],
                   "N": n, "NT": nt, "xi": cfg.xi, "rc": cfg.rc, "M": cfg.M, "P": cfg.P,
                   "Mtilde": cfg.Mtilde, "fft_grid": cfg.D,
                   "eta": round(cfg.eta, 4),
                   "parallelism": (f"replicas x{dist.world}" if dist.world > 1
                                   else "one GPU, the whole evaluation"),
                   "l2": working_set_note(w, cfg),
                   "green_precompute_s": round(precompute_s, 3)},
        "e2e": {"value": nt * e2e_steps * dist.world / e2e_s, "unit": "targets/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "api": "fse_cuda_total_sum (host buffers, pinned in and out)"},
        "roofline": roof,
        "stage_roofline": stage_roof,
        "stage_ms": {k: round(v, 4) for k, v in stage_ms.items()},
        "stage_timings_s": {k: v / nbrk for k, v in tm.as_dict().items()},
        "realspace_work": {"candidates": int(rs_cand), "pairs": int(rs_pairs),
                           "pair_flops": PAIR_FLOPS[w["kind"]]},
        "gpu_launches": int(launches),
        "gpu_launches_note": "our kernels (cuFFT library launches not counted)",
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    if dist.rank == 0:
        emit(line)
    for p in (d_pos, d_str, d_u) + (() if tas else (d_tgt,)):
        ctx.dev_free(p)


def traffic_for(workload: str, kernel: str):
    """dram read+write bytes per launch of `kernel` at `workload` from the committed
    ncu --set full capture (profiles/traffic.json, keyed by workload), else None."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        t = json.load(f)
    return (t.get(workload) or {}).get(kernel)


def working_set_note(w, cfg):
    """Bytes the Fourier part streams per step vs the 126 MB L2."""
    a = 9 if w["kind"] == 1 else 3
    D, Mt = cfg.D, cfg.Mtilde
    Dh = D // 2 + 1
    ws = a * (8 * Mt ** 3 + 16 * Mt * Mt * Dh + 16 * Mt * D * Dh) + 8 * D * D * Dh
    ws += w["n"] * (24 + 8 * a + 24 * cfg.P)
    gb = ws / 1e9
    if ws > 8 * 126e6:
        return f"working set ~{gb:.2f} GB >> 126 MB L2 (inputs larger than L2): no flush needed"
    return (f"working set ~{gb:.2f} GB, not >> 126 MB L2: part of it may stay L2-resident "
            "between steps (no explicit flush)")


# ------------------------------------------------------------------ reference CPU
def _avail_bytes():
    try:
        import psutil
        return psutil.virtual_memory().available
    except Exception:
        return 16 << 30


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_full(w, steps: int, warmup: int, budget_s: float):
    """Time the UNMODIFIED reference fse::total_sum (oracle/_ref: /root/reference
    sources compiled by oracle/Makefile, OpenMP) on this host at the full workload.
    Inputs from the reference-side generator (oracle/ref_capi.cpp), the Green's
    table from the reference's own precompute_mollified_green (excluded from the
    timing, as harness.hpp:50 does).  `warmup` untimed calls, then timed calls
    until `steps` are done or `budget_s` of timed calls has elapsed (>= 1).
    Threads: every host thread, capped so the reference's memory (a private
    Mtilde^3 spread grid per thread, ewald.cpp:166-176, plus the C2C spectra)
    fits in 85 % of available RAM.  Returns (result dict, None) or (None, why)."""
    from oracle import refimpl as R
    if not R.available():
        return None, "oracle/_ref (the reference built from its sources) is missing"
    pos, st, tgt = R.generate_workload(w["wl"], w["n"], SEED)
    cfg = workload_config(w, st, R)
    a = 9 if w["kind"] == 1 else 3
    D, Mt = cfg.D, cfg.Mtilde
    fixed = a * 8 * Mt ** 3 + (a + 3) * 16 * D ** 3 + 8 * D ** 3 + w["n"] * (48 + 8 * a) * 3
    per_thread = a * 8 * Mt ** 3
    avail = 0.85 * _avail_bytes()
    cores = os.cpu_count() or 1
    thr = min(cores, int((avail - fixed) // per_thread)) if avail > fixed else 0
    if thr < 1:
        return None, (f"reference total_sum needs ~{(fixed + per_thread) / 1e9:.0f} GB of host "
                      f"RAM; {avail / 0.85 / 1e9:.0f} GB available")
    R.set_threads(thr)
    targets = pos if tgt is None else tgt
    t0 = time.perf_counter()
    green = R.precompute_green(R.green_kind_for(w["kind"]), cfg.Ltilde, cfg.Mtilde, cfg.sf)
    pre_s = time.perf_counter() - t0
    times, stages = [], []
    i = 0
    while True:
        tm = {}
        t0 = time.perf_counter()
        R.total_sum(cfg, w["kind"], pos, st, targets, green, timings=tm)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
            stages.append(tm)
        i += 1
        if i >= warmup + steps or (times and sum(times) >= budget_s):
            break
    med = float(np.median(times))
    keys = ("spread", "fft", "scale", "quadrature", "realspace", "total")
    st_med = {k: float(np.median([s[k] for s in stages])) for k in keys}
    return {"seconds": times, "median_s": med, "threads": thr, "cores": cores,
            "cpu": _cpu_model(), "precompute_s": pre_s, "stages_s": st_med,
            "warmup": min(warmup, i), "nt": targets.shape[0]}, None


REF_NOTE = ("the reference's own sources (oracle/_ref, g++ -O2 -fopenmp), FFTs through "
            "oracle/fftw_shim (FFTW3 is absent; the shim is OpenMP-parallel over 1D lines, "
            "i.e. faster than the reference's single-threaded FFTW as written, fft.cpp)")


def cpu_baseline_line(w):
    r, why = reference_full(w, steps=1, warmup=0, budget_s=0.0)
    if r is None:
        return {"value": None, "unit": "targets/s", "cores": 0, "kind": "reference",
                "sample": f"not run: {why}"}
    return {"value": r["nt"] / r["median_s"], "unit": "targets/s", "cores": r["threads"],
            "kind": "reference",
            "sample": (f"one full fse::total_sum call at the bench workload ({w['desc']}), "
                       f"no sub-sampling or extrapolation; {REF_NOTE}; {r['threads']} OpenMP "
                       f"threads of {r['cores']} ({r['cpu']}); Green's precompute "
                       f"({r['precompute_s']:.1f} s) excluded as harness.hpp:50 does"),
            "seconds": r["median_s"], "stages_s": r["stages_s"]}


def run_reference(args):
    """--impl reference: rank 0 only (other torchrun ranks exit 0 without work)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    w = WORKLOADS[args.workload]
    r, why = reference_full(w, steps=max(1, args.steps), warmup=min(args.warmup, 1),
                            budget_s=args.ref_budget_s)
    if r is None:
        emit({"impl": "reference", "unavailable": why})
        return
    v = r["nt"] / r["median_s"]
    line = {
        "impl": "reference", "metric": metric_name(w), "value": v, "unit": "targets/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": len(r["seconds"]),
        "warmup": r["warmup"], "ms_per_step": r["median_s"] * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: SURVEY 8(d) generator {w['wl']} (seed {SEED}), reference-side "
                "generator (oracle/ref_capi.cpp), no dataset",
        "config": {"workload": f"{args.workload}: {w['desc']}", "kind": KIND_NAMES[w["kind"]],
                   "N": w["n"], "NT": r["nt"], "parallelism": "host CPU (OpenMP), rank 0 only",
                   "steps_requested": args.steps, "warmup_requested": args.warmup,
                   "step_note": (f"timed calls stop at {args.steps} or once {args.ref_budget_s:.0f} s "
                                 "of timed calls have elapsed; ms_per_step = median of the "
                                 "timed calls, each a full-size call (no extrapolation)"),
                   "seconds_per_call": [round(x, 3) for x in r["seconds"]],
                   "product_library_loaded": _product_loaded()},
        "cpu_baseline": {"value": v, "unit": "targets/s", "cores": r["threads"],
                         "kind": "reference",
                         "sample": (f"full fse::total_sum calls at the bench workload; {REF_NOTE}; "
                                    f"{r['threads']} OpenMP threads of {r['cores']} ({r['cpu']}); "
                                    f"Green's precompute ({r['precompute_s']:.1f} s) excluded"),
                         "stages_s": r["stages_s"]},
        "e2e": {"value": v, "unit": "targets/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)


def _product_loaded() -> bool:
    """Whether this process mapped libfse_b200.so (the reference arm must not)."""
    try:
        with open("/proc/self/maps") as f:
            return "libfse_b200" in f.read()
    except OSError:
        return False


def relaunch_under_torchrun(n: int) -> int:
    """`python bench.py --gpus N` without torchrun: run N ranks on this node."""
    port = os.environ.get("MASTER_PORT", "29533")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", port, os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent full evaluations per GPU instead of z-slabs")
    ap.add_argument("--slabs", action="store_true",
                    help="use the partitioned path also at N = 1 (one slab, NCCL group of one)")
    ap.add_argument("--ref-budget-s", type=float, default=80.0,
                    help="--impl reference: stop timing full-size calls after this many seconds")
    ap.add_argument("--fp64-peak", type=float, default=None,
                    help="TFLOP/s; default: measured in-run with a DFMA loop")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    _stdout_to_stderr()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    dist = Dist(force_group=args.slabs and args.impl == "ours")
    try:
        if (dist.world > 1 and not args.replicas) or args.slabs:
            run_dist(args, dist)
        else:
            run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
