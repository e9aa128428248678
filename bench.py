#!/usr/bin/env python3
"""Benchmark: MPM particle-substeps/s, forward+backward, on the 1M-particle multi-material scene.

One "step" = one grad_trajectory (grad.hpp:61-134) over the full horizon of the
scene (10 segments x 50 substeps): T forward substeps, a target-point loss per
segment, and T adjoint substeps producing the action gradient.
value = active particles * T / device time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1: the c4 scooping scene (1,027,233 particles of
water + an elastic floater on a 128^3 grid, a three-box ladle effector), the
1M-particle multi-material scene the north star's single-GPU target names.
The same line carries `configs` (c1, c2, c3 on one GPU, one segment each; c5 over
SCALE_HORIZON) and `scaling_base` (c5 on one GPU over the same horizon as N > 1).
N > 1 (torchrun, one process per GPU): the north star's scaling scene c5
(8,044,544 particles, 256^3) split into x-slabs, one per GPU:
halo planes and migrating particles go to the neighbouring ranks (CUDA IPC peer
copies into exported device inboxes over NVLink by default, `--transport nccl` for NCCL),
rigid/loss/effector sums are all-reduced, so the scaling is strong (compare
with `scaling_base` of the N = 1 line).  If the slab transport cannot start the
run prints an `error` line and exits non-zero (no silent fallback).
The reference arm (--impl reference) times the unmodified reference engine
(oracle/_ref, proj/include/flume compiled as-is) on this host's CPU cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MPM particle-substeps/sec fwd & fwd+bwd at 1/2/4/8 B200; HBM GB/s vs peak"
UNIT = "particle-substeps/s"
SCENE = "c4"        # N = 1
SCENE_SCALE = "c5"  # N > 1: the 8M-particle 256^3 slab-partitioned scene
HORIZON = 500  # c4's full horizon: optimizer.n_segments (10) x segment_length (50)
# c5 at 256^3 is a valid simulation for ~30 substeps only: its jelly's P-wave crosses 1.2 cells
# per substep, so the explicit scheme diverges and the reference itself raises
# DegenerateDeformation before substep 100 (profiles/r02_c5_stability.json, the unmodified
# reference and the device agree).  The scaling workload therefore stays inside that window.
SCALE_HORIZON = 20

# algorithmic bytes per launch unit: fp32 state, each
# field counted once per kernel that must move it; N = active particles, A =
# touched nodes (64 per node block)
KERNELS = ["p2g", "grid_update", "g2p", "sort", "g2p_adjoint", "grid_adjoint", "p2g_adjoint", "rigid", "other",
           "slab_comm"]
ALG_BYTES = {
    "p2g": (100, 16),           # read x v F C class | write m,p per node
    "grid_update": (0, 44),     # read m,p (16) write v,m (16) + v0,m (16) - forward writes only v: use 44 avg
    "g2p": (148, 16),           # read x F class, write x v F C | read v,m per node
    "g2p_adjoint": (196, 32),   # read x F class + 4 bars, write x_bar F_bar | read v, write v_bar
    "grid_adjoint": (0, 48),
    "p2g_adjoint": (244, 16),   # read x v F C class + x_bar F_bar, write 4 bars | read m_bar,p_bar
}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region
    (one nvidia-smi process in loop mode, -lms 50)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self._p = None
        self._t = None

    def _reader(self):
        for line in self._p.stdout:
            f = [s.strip() for s in line.strip().split(",")]
            if len(f) == 6:
                self.samples.append((time.perf_counter(), f))

    def mark(self, which):
        setattr(self, "t_" + which, time.perf_counter())

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "50"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._reader, daemon=True)
            self._t.start()
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is not None:
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
        if self._t:
            self._t.join(timeout=5)

    def summary(self):
        """Samples that arrived inside the timed window (marks 'start'/'end'); if the
        window was shorter than the sampling period, the ones within 0.25 s of it."""
        t0, t1 = getattr(self, "t_start", 0.0), getattr(self, "t_end", 1e30)
        win = [f for t, f in self.samples if t0 <= t <= t1 + 0.06]
        near = win or [f for t, f in self.samples if t0 - 0.25 <= t <= t1 + 0.25]
        if not near:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in near if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in near if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in near for k in range(4) if s[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(near), "samples_in_window": len(win)}


def cpu_reference_sample(scene: str = SCENE, substeps: int = 4, stride: int = 2):
    """The reference engine (oracle/_ref) on this host, single-threaded like the reference:
    grad_trajectory over `substeps` substeps of the same scene (SURVEY.md 8(d) protocol)."""
    from oracle import ref
    from paper_2303_02346_b200 import scenes
    spec = scenes.load(scene)
    r = ref.RefWorld(spec)
    init = np.array(spec["optimizer"]["init"], dtype=np.float64)
    t0 = time.perf_counter()
    r.grad_trajectory(init.reshape(1, 6), substeps, stride=stride)
    dt = time.perf_counter() - t0
    return r.n * substeps / dt, r.n, dt


def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref = proj/include compiled unmodified)
    on this box's host cores.  The reference engine is single-threaded per scene, so it uses
    every host thread the only way it can: one independent replica of the workload per
    thread (ctypes releases the GIL), bounded by host memory.  A step = every replica runs
    one bounded sample (grad_trajectory over `sub` substeps, stride 1); value = aggregate
    particle-substeps / wall time."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor

    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libflume_ref.so not built"}))
        return
    from paper_2303_02346_b200 import scenes
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 64e9
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    world_size = int(os.environ.get("WORLD_SIZE", "1"))
    scene = args.scene or (SCENE if world_size == 1 else SCENE_SCALE)  # the same workload as our arm
    spec = scenes.load(scene)
    # a replica holds the AoS state (224 B/particle) ~4 times over (state, capture, cache) plus
    # the 56 B/node grid; c4 ~1.1 GB, c5 ~8.2 GB -- keep 2x headroom
    res = spec["grid_resolution"]
    per_rep = 2 * (4 * 224 * 1.03e6 * (res / 128) ** 3 + 56 * (res + 1) ** 3)
    reps = max(1, min(threads, int(avail // per_rep)))
    init = np.array(spec["optimizer"]["init"], dtype=np.float64).reshape(1, 6)
    sub = 1  # one forward + adjoint substep per replica per step keeps K + W steps within minutes
    with ThreadPoolExecutor(reps) as pool:
        worlds = list(pool.map(lambda _: ref.RefWorld(spec), range(reps)))
        n = worlds[0].n

        def sample(r):
            r.grad_trajectory(init, sub, stride=1)

        for _ in range(args.warmup):
            list(pool.map(sample, worlds))
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            list(pool.map(sample, worlds))
            times.append(time.perf_counter() - t0)
    total_t = sum(times)
    value = reps * n * sub * args.steps / total_t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{scenes.NAMES[scene]} grad_trajectory, {sub}-substep sample per step per "
                                   f"replica, stride 1; {reps} independent replicas, one per host thread",
                       "particles": n, "grid": f"{res}^3", "replicas": reps},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": reps, "kind": "reference",
                             "sample": f"grad_trajectory over {sub} substeps of {scene} per replica per step "
                                       f"({reps} threads, g++ -O3 build of proj/include)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def _watchdog(seconds: float, rank: int):
    """A multi-process run that stops making progress is ended with a JSON line, not a hang."""
    def bite():
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT,
                              "error": f"watchdog: no result after {seconds:.0f} s"}), flush=True)
        os._exit(3)
    t = threading.Timer(seconds, bite)
    t.daemon = True
    t.start()


def _device_ms(lib, ctx, check, fn, slot0=6):
    """Device time of fn() on the context stream (CUDA events on that stream)."""
    import ctypes as C
    check(lib.flume_timer_mark(ctx, slot0))
    fn()
    check(lib.flume_timer_mark(ctx, slot0 + 1))
    ms = C.c_double()
    check(lib.flume_timer_elapsed(ctx, slot0, slot0 + 1, C.byref(ms)))
    return ms.value


def _stride_for(fl, w, T, seglen, n_local, device, sharing=1):
    """The whole trajectory in HBM (stride = horizon) keeps per substep the state and its
    permutation (~124 B per particle), the recorded grid (two dense float4 node arrays and
    a contact mask, ~33 B per node of the block-major grid) and the block lists with their
    work order (~128 B per block); where the device cannot hold it the backward replays from
    checkpoints at segment boundaries (CheckpointStore stride)."""
    import torch
    try:
        free_b = torch.cuda.mem_get_info(device)[0]
    except Exception:
        free_b = 0
    nb_tot = 1
    for d in w.scene.node_dims:
        nb_tot *= (d + 3) // 4
    need = sharing * T * (n_local * 124 + (33 * 64 + 128) * nb_tot) * 1.15
    return (T if (free_b == 0 or free_b > need) else seglen), free_b, need


def scene_rates(name, steps, warmup, horizon=None, device=0):
    """One-GPU fwd and fwd+bwd rates of a BASELINE config (device time, CUDA events): fwd+bwd =
    grad_trajectory over `horizon` substeps (default one optimizer segment), fwd = the same
    number of mpm_substep calls from the uploaded state (re-uploaded, untimed, every step)."""
    import paper_2303_02346_b200 as fl
    from paper_2303_02346_b200 import scenes
    w = fl.build_scene(scenes.load(name))
    ws = fl.GpuWorkspace(w.scene, device=device)
    lib, ctx = ws.lib, ws.ctx
    check = lambda rc: fl.api._raise(lib, ctx, rc)  # noqa: E731
    n = int(np.sum(w.scene.activation_substep <= 0))
    seglen = w.segment_length or 50
    T = horizon or seglen
    nseg = max(1, T // seglen)
    seglen = T // nseg
    acts = fl.ActionTrajectory(nseg, seglen, np.tile(w.init_action.reshape(1, 6), (nseg, 1)))
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    stride, _, _ = _stride_for(fl, w, T, seglen, n, device)
    for _ in range(warmup):
        fl.grad_trajectory(w.scene, w.state, acts, loss, stride=stride, ws=ws)
    gms = 0.0
    for _ in range(steps):
        g = fl.grad_trajectory(w.scene, w.state, acts, loss, stride=stride, ws=ws)
        gms += g.forward_ms + g.backward_ms
    fms = 0.0
    for _ in range(steps):
        st = w.state.copy()
        ws._upload(st)
        fms += _device_ms(lib, ctx, check, lambda: check(lib.flume_substep(ctx, fl.api._dp(w.init_action), T)))
    out = {"particles": n, "grid": f"{w.scene.grid_resolution}^3", "substeps": T, "stride": stride,
           "fwd_bwd": n * T * steps / (gms / 1e3), "fwd": n * T * steps / (fms / 1e3),
           "fwd_bwd_ms_per_substep": gms / steps / T, "fwd_ms_per_substep": fms / steps / T}
    ws.close()
    return out


def population_rates(name, R, steps, warmup, device=0):
    """A population of R candidates of a BASELINE config in one replica context (SURVEY.md
    8(f)3): fwd+bwd = grad_trajectory_replicas over one optimizer segment, fwd = the same
    substeps of all R (device time, CUDA events); rates count all R candidates' particles."""
    import paper_2303_02346_b200 as fl
    from paper_2303_02346_b200 import scenes
    w = fl.build_scene(scenes.load(name))
    rws = fl.ReplicaWorkspace(w.scene, R, device=device)
    lib, ctx = rws.lib, rws.ctx
    check = lambda rc: fl.api._raise(lib, ctx, rc)  # noqa: E731
    n = int(np.sum(w.scene.activation_substep <= 0))
    T = w.segment_length or 50
    rng = np.random.default_rng(0)
    pop = [fl.ActionTrajectory(1, T, w.init_action.reshape(1, 6) + 0.1 * rng.standard_normal((1, 6)))
           for _ in range(R)]
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    for _ in range(warmup):
        fl.grad_trajectory_replicas(w.scene, w.state, pop, loss, rws)
    gms = 0.0
    for _ in range(steps):
        g = fl.grad_trajectory_replicas(w.scene, w.state, pop, loss, rws)
        gms += g[0].forward_ms + g[0].backward_ms
    acts = np.ascontiguousarray(np.concatenate([a.values[0] for a in pop]))
    fms = 0.0
    for _ in range(steps):
        rws._upload(rws.replicate(w.state))
        fms += _device_ms(lib, ctx, check, lambda: check(lib.flume_substep(ctx, fl.api._dp(acts), T)))
    out = {"replicas": R, "particles": R * n, "substeps": T, "fwd_bwd": R * n * T * steps / (gms / 1e3),
           "fwd": R * n * T * steps / (fms / 1e3), "context": "one replica context: every launch covers all R"}
    rws.close()
    return out


def run_ours(args):
    import ctypes as C

    import paper_2303_02346_b200 as fl
    from paper_2303_02346_b200 import _abi, scenes
    from paper_2303_02346_b200.api import _dp

    world_size = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    import torch
    if world_size > 1:
        import torch.distributed as dist
        # (more ranks than visible GPUs only happens when the launcher is exercised on a
        # small box; the ranks then share devices)
        local = local % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local)
        # torch.distributed is host plumbing only (id broadcast, barriers, max-over-ranks
        # timings): gloo; the data path between the GPUs is the library's own transport
        # (CUDA IPC peer copies over NVLink, or NCCL with --transport nccl)
        dist.init_process_group("gloo")
        _watchdog(args.deadline, rank)

    scene_name = args.scene or (SCENE if world_size == 1 else SCENE_SCALE)
    spec = scenes.load(scene_name)
    w = fl.build_scene(spec)
    lib = _abi.load()
    mode = "single"
    ws = None
    if world_size > 1:
        obj = [None]
        if rank == 0:
            try:
                obj[0] = fl.ipc_unique_id() if args.transport == "ipc" else fl.dist_unique_id()
            except Exception as e:
                obj[0] = "error: " + str(e)
        dist.broadcast_object_list(obj, src=0)
        err = None
        if isinstance(obj[0], bytes):
            try:
                ws = fl.GpuWorkspace.distributed(w.scene, local, rank, world_size, obj[0])
                mode = "slabs"
            except Exception as e:
                err = str(e)
        else:
            err = obj[0]
        ok = torch.tensor([1 if mode == "slabs" else 0])
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            if rank == 0:
                print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world_size,
                                  "error": f"x-slab {args.transport} transport did not start: "
                                           f"{err or 'failed on a peer rank'}"}),
                      flush=True)
            os._exit(4)
    if ws is None:
        ws = fl.GpuWorkspace(w.scene, device=local)
    ctx = ws.ctx
    n = int(np.sum(w.scene.activation_substep <= 0))
    T = args.horizon or (HORIZON if world_size == 1 else SCALE_HORIZON)
    seglen = min(w.segment_length or T, T)
    if T % seglen:
        seglen = T
    nseg = T // seglen
    acts = fl.ActionTrajectory(nseg, seglen, np.tile(w.init_action.reshape(1, 6), (nseg, 1)))
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)

    # pinned host copies of the inputs for the end-to-end leg
    pin = {k: torch.empty(getattr(w.state, k).shape, dtype=torch.float64).pin_memory()
           for k in ("x", "v", "F", "C")}
    for k in pin:
        pin[k].numpy()[...] = getattr(w.state, k)
    effs = fl.GpuWorkspace._eff_to_c(w.state.effectors)
    view = _abi.StateView()
    view.time, view.substep_index = 0.0, 0
    view.x, view.v = (C.cast(pin["x"].data_ptr(), C.POINTER(C.c_double)),
                      C.cast(pin["v"].data_ptr(), C.POINTER(C.c_double)))
    view.F, view.C = (C.cast(pin["F"].data_ptr(), C.POINTER(C.c_double)),
                      C.cast(pin["C"].data_ptr(), C.POINTER(C.c_double)))
    view.effectors = effs
    h2d = sum(pin[k].numel() * 8 for k in pin)
    a_c = acts._c()
    grad = np.zeros((nseg, 6))
    lo, fu, snaps = C.c_double(), C.c_double(), C.c_long()
    per = np.zeros(nseg)

    def check(rc):
        fl.api._raise(lib, ctx, rc)

    def upload():
        check(lib.flume_state_upload(ctx, C.byref(view)))

    sharing = max(1, -(-world_size // max(torch.cuda.device_count(), 1)))  # ranks per device
    per_rank_n = n / world_size if mode == "slabs" else n
    stride, free_b, need = _stride_for(fl, w, T, seglen, per_rank_n, local, sharing)
    print(f"[bench rank {rank}] {scene_name}: free {free_b / 1e9:.1f} GB, whole-trajectory estimate "
          f"{need / 1e9:.1f} GB -> checkpoint stride {stride}", file=sys.stderr, flush=True)

    def step():
        check(lib.flume_grad_trajectory(ctx, C.byref(a_c), C.byref(loss.desc), stride, 0, _dp(grad), C.byref(lo),
                                        C.byref(fu), _dp(per), C.byref(snaps)))

    def fwd_only():
        check(lib.flume_substep(ctx, _dp(w.init_action), T))

    def max_over_ranks(v):
        if not dist:
            return v
        tt = torch.tensor([v])
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    upload()
    # the clock sampler runs from the warm-up on; its summary keeps the samples
    # that arrived inside the timed window
    with ClockSampler(local) as clocks:
        for _ in range(args.warmup):
            step()
        if dist:
            dist.barrier()
        check(lib.flume_sync(ctx))

        # ---- timed: device time over exactly K steps (inputs resident in HBM) ----
        launches = 0
        fwd_ms = bwd_ms = 0.0
        clocks.mark("start")
        check(lib.flume_timer_mark(ctx, 0))
        for _ in range(args.steps):
            step()  # synchronous: returns the loss and gradient in host memory
            t = ws.last_timing()
            launches += t.launches
            fwd_ms += t.forward_ms
            bwd_ms += t.backward_ms
        check(lib.flume_timer_mark(ctx, 1))
        ms = C.c_double()
        check(lib.flume_timer_elapsed(ctx, 0, 1, C.byref(ms)))
        clocks.mark("end")
        if dist:
            dist.barrier()
    total_ms = max_over_ranks(ms.value)
    # ---- per-kernel CUDA-event times: a separate instrumented pass of the same K steps
    #      (event bookkeeping on the host would otherwise perturb the timed region) ----
    check(lib.flume_profile(ctx, 1))
    for _ in range(args.steps):
        step()
    kms = (C.c_double * len(KERNELS))()
    kcnt = (C.c_long * len(KERNELS))()
    check(lib.flume_kernel_times(ctx, kms, kcnt, len(KERNELS)))
    check(lib.flume_profile(ctx, 0))
    value = n * T * args.steps / (total_ms / 1e3)

    # ---- forward-only rate (mpm_substep chain over the same horizon from the same
    #      uploaded state: re-uploaded before every step, outside the timed events) ----
    fwd_ms_all = 0.0
    for _ in range(args.steps):
        upload()
        fwd_ms_all += _device_ms(lib, ctx, check, fwd_only, 2)
    fwd_ms_all = max_over_ranks(fwd_ms_all)
    fwd_value = n * T * args.steps / (fwd_ms_all / 1e3)

    # ---- end to end through the public C ABI: H2D of the state from pinned host
    #      memory, grad_trajectory, D2H of loss + action gradient, every step ----
    if dist:
        dist.barrier()
    check(lib.flume_timer_mark(ctx, 4))
    for _ in range(args.steps):
        upload()
        step()  # returns loss/gradient in host memory (D2H inside)
    check(lib.flume_timer_mark(ctx, 5))
    ems = C.c_double()
    check(lib.flume_timer_elapsed(ctx, 4, 5, C.byref(ems)))
    e2e_ms = max_over_ranks(ems.value)
    e2e_value = n * T * args.steps / (e2e_ms / 1e3)
    # slabs: rank 0's share of the work, for its roofline line
    keys, ids, na, _ = ws.store_order(w.state)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel class ----
    peak, peak_kind = peaks()
    nb_nodes = None
    kern = {}
    for i, name in enumerate(KERNELS):
        if kcnt[i]:
            kern[name] = {"ms_total": kms[i], "launches": int(kcnt[i]), "us_per_launch": 1e3 * kms[i] / kcnt[i]}
    dom = max((k for k in kern if k in ALG_BYTES), key=lambda k: kern[k]["ms_total"])
    # active nodes per substep: touched node blocks x 64 (measured on the first step's lists)
    A = int(0.155 * n * 1.6)  # fallback estimate; replaced by the measured value below
    n_local = int(na)
    try:
        blocks = np.unique(keys[:na] >> 6)
        nd = w.scene.node_dims
        NB = [(d + 3) // 4 for d in nd]
        bz = blocks % NB[2]
        by = (blocks // NB[2]) % NB[1]
        bx = blocks // (NB[2] * NB[1])
        touched = set()
        for dxx in (0, 1):
            for dyy in (0, 1):
                for dzz in (0, 1):
                    touched.update(((bx + dxx) * NB[1] + by + dyy) * NB[2] + bz + dzz)
        A = 64 * len(touched)
    except Exception:
        pass
    pb, nb = ALG_BYTES[dom]
    alg = pb * n_local + nb * A
    per_launch_s = kern[dom]["ms_total"] / kern[dom]["launches"] / 1e3
    achieved = alg / per_launch_s / 1e9
    traffic = None
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(dom)
        except Exception:
            traffic = None

    # the same figures for every kernel class with algorithmic bytes (P2G / G2P are the
    # north star's ">= 50% of HBM roofline" kernels); traffic = ncu DRAM bytes per launch
    per_kernel = {}
    try:
        tr_all = json.loads(prof.read_text()) if prof.exists() else {}
    except Exception:
        tr_all = {}
    for k, (pbk, nbk) in ALG_BYTES.items():
        if k not in kern:
            continue
        t_s = kern[k]["ms_total"] / kern[k]["launches"] / 1e3
        a_k = (pbk * n_local + nbk * A) / t_s / 1e9
        tk = tr_all.get(k)
        per_kernel[k] = {"achieved": a_k, "frac": a_k / peak, "us_per_launch": 1e6 * t_s,
                         "alg_bytes_per_launch": pbk * n_local + nbk * A, "traffic": tk,
                         "traffic_frac": (tk / t_s / 1e9 / peak) if tk else None}

    cpu = None
    if not args.no_cpu and world_size == 1:
        try:
            rate, rn, dt = cpu_reference_sample(scene_name, 4, 2)
            cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"reference grad_trajectory, {scene_name} ({rn} particles), 4 substeps, stride 2, "
                             f"{dt:.1f} s on 1 host core (g++ -O3 build of proj/include)"}
        except Exception as e:  # keep the GPU line even if the host leg fails
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": f"failed: {e}"}

    # ---- the other BASELINE configs on this GPU (one optimizer segment each), and the
    #      strong-scaling base: the N > 1 workload (c5, SCALE_HORIZON substeps) on one GPU ----
    configs, scaling_base = {}, None
    if world_size == 1 and not args.no_configs:
        ws.close()
        for name in ("c1", "c2", "c3", "c5"):
            try:
                configs[name] = scene_rates(name, 2, 1, horizon=SCALE_HORIZON if name == SCENE_SCALE else None,
                                            device=local)
            except Exception as e:
                configs[name] = {"error": str(e)}
        try:  # a CMA-ES-sized population of the small scene in one replica context
            configs["c1x16"] = population_rates("c1", 16, 2, 1, device=local)
        except Exception as e:
            configs["c1x16"] = {"error": str(e)}
        try:
            sb = scene_rates(SCENE_SCALE, 2, 1, horizon=SCALE_HORIZON, device=local)
            scaling_base = {"scene": SCENE_SCALE, "value": sb["fwd_bwd"], "fwd": sb["fwd"], "unit": UNIT,
                            "particles": sb["particles"], "horizon": SCALE_HORIZON, "stride": sb["stride"],
                            "note": "bench.py --gpus N>1 runs this workload as x-slabs; strong-scaling "
                                    "efficiency(N) = value(N) / (N * this value)"}
        except Exception as e:
            scaling_base = {"scene": SCENE_SCALE, "error": str(e)}

    grid = f"{w.scene.grid_resolution}^3"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world_size, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if mode == "slabs" else "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": f"synthetic: reference scene JSON {scene_name} (SURVEY.md App. A) sampled by the reference "
                "lattice+jitter rule",
        "config": {"workload": f"{scenes.NAMES[scene_name]}: grad_trajectory over " + (
                               "the full horizon" if T == HORIZON else f"{T} substeps (the scene's stable window)") +
                               f", {nseg} "
                               f"segments x {seglen} substeps, stride {stride} " + (
                                   "(forward + adjoint, the whole trajectory kept in HBM: no checkpoint replay)"
                                   if stride == T else
                                   "(forward + adjoint, checkpoints at segment boundaries: the backward "
                                   "replays each segment, the device could not hold the whole trajectory)") +
                               ", target_point loss per segment",
                   "particles": n, "grid": grid, "active_nodes": A, "horizon": T,
                   "l2": "inputs larger than L2 (trajectory store ~%.1f GB per step)" % (n * 112 * (T + 1) / 1e9),
                   "parallelism": "single" if mode == "single" else
                   f"x-slabs over {world_size} GPUs ({'CUDA IPC' if args.transport == 'ipc' else 'NCCL'} halos "
                   "and migration)",
                   **({"rank0_particles": n_local} if mode == "slabs" else {})},
        "fwd": {"value": fwd_value, "unit": UNIT,
                "workload": f"mpm_substep x {T} from the uploaded state (re-uploaded untimed every step)"},
        "fwd_bwd_split_ms": {"forward": fwd_ms / args.steps, "backward": bwd_ms / args.steps},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d * world_size,
                "d2h_bytes_per_step": 8 * (7 * nseg + 2) * world_size},  # gradient, per-segment and total losses
        "gpu_launches": int(launches),
        "kernels": kern,
        "roofline": {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "alg_bytes_per_launch": alg},
        "roofline_by_kernel": per_kernel,
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
        **({"configs": configs} if configs else {}),
        **({"scaling_base": scaling_base} if scaling_base else {}),
    }
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--horizon", type=int, default=None,
                    help=f"substeps per step (default {HORIZON} for c4 at N = 1, {SCALE_HORIZON} for c5 at N > 1)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config and scaling-base legs")
    ap.add_argument("--scene", default=None, help="override the scene (c1..c5)")
    ap.add_argument("--deadline", type=float, default=600.0, help="multi-GPU watchdog (s)")
    ap.add_argument("--transport", default="ipc", choices=["ipc", "nccl"],
                    help="x-slab data path for N > 1: CUDA IPC peer copies (default) or NCCL")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
