#!/usr/bin/env python
"""Benchmark: DRRs/sec fwd+bwd (200x200 detector, 512x512x133 CT) on B200.

One STEP = the hot path over one fixed global batch of poses (default 256):
for every pose, render the 200x200 DRR, evaluate the reference's registration
loss (neg-ZNCC vs a fixed DRR, metrics.py:71-91) and back-propagate to the
pose -- the reference's ``loss_and_gradient`` (gradients.py:61-69) for each
pose, config C2 of SURVEY.md 8(d) with the C4 pose sampling.  On N GPUs the
batch is sharded over the ranks (strong scaling: the work per step is fixed):
each rank walks its block of poses and its kernels store the per-pose loss and
7-gradient straight into rank 0's buffers over NVLink
(distributed.ShardedDRR); the CT is NCCL-broadcast once before timing.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]

Prints ONE JSON line (rank 0).  Timing: CUDA events per step on the launching
stream, L2 flushed (256 MiB write) between timed steps outside the events,
max over ranks.  Also measured (rank 0's line, keys below): the same step
end to end (pinned host poses in, loss + gradient back on the host), the C1 /
C4 / C5 configs, C3 registration, the dominant kernel against the HBM
roofline, and the reference's CPU path on this host.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SPACING = (0.703125, 0.703125, 2.5)
DIMS = (512, 512, 133)
H = W = 200
PITCH = 3.6
RHO = 300.0
TRUTH = (RHO, math.pi / 2, math.pi / 2, 0.0, 0.0, 0.0, 0.0)
METRIC = "DRRs/sec fwd+bwd (200x200 det, 512x512x133 CT)"
WORKLOAD = ("C2: synthetic chest CT 512x512x133 @ (0.703125,0.703125,2.5) mm fp32, "
            "200x200 detector @ 3.6 mm, rho=sdr=300 mm; per step a fixed global batch of poses "
            "(narrow samples around AP, seed 0) x [forward DRR + neg-ZNCC vs fixed DRR at the "
            "truth pose + backward to (rho, rotation, translation)], sharded over the GPUs, "
            "per-pose loss and gradient collected on rank 0")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--batch", type=int, default=256, help="global poses per step (all GPUs)")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-other-configs", action="store_true",
                   help="skip the C1/C3/C4/C5 context measurements")
    p.add_argument("--cpu-seconds", type=float, default=15.0,
                   help="wall-time budget of the CPU-baseline sample")
    return p.parse_args()


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.5)  # nvidia-smi start-up: sample before the timed region begins
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in getattr(self, "lines", []):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ CPU baseline
# The reference's own CPU path: drrtrace's loss_and_gradient with its native
# (Cython, single-threaded, GIL-holding) backend from oracle/_ref, one pose per
# call, pose-sharded over a fork pool created ONCE (outside any timed region).
_REF_STATE = {}


def _ref_worker(eta):
    from oracle.oracle import reference_module
    dt = reference_module()
    st = _REF_STATE
    t0 = time.perf_counter()
    rec = dt.loss_and_gradient(st["vol"], dt.PoseParameters.from_vector(eta), st["spec"],
                               st["fixed"], "neg_zncc", backend="native")
    return time.perf_counter() - t0, float(rec.value)


def _port_worker(eta):
    """Fallback when oracle/_ref is absent: the C oracle (port) fwd + bwd."""
    from oracle import oracle as O
    st = _REF_STATE
    t0 = time.perf_counter()
    frame = O.pose_frame(eta, st["center"])
    img = O.render(st["flat"], DIMS, SPACING, (0, 0, 0), frame, H, W, PITCH, PITCH)
    val, pg = O.neg_zncc_value_and_grad(img, st["fixed"])
    O.render_backward(st["flat"], DIMS, SPACING, (0, 0, 0), frame, H, W, PITCH, PITCH, pg)
    return time.perf_counter() - t0, float(val)


def cpu_setup(vol_np):
    """Reference inputs: the fp32 CT cast back to f64 (the GPU arm's values)."""
    from oracle.oracle import reference_module
    dt = reference_module()
    flat = vol_np.astype(np.float64).ravel(order="F")
    center = tuple(0.5 * n * s for n, s in zip(DIMS, SPACING))
    _REF_STATE.update(flat=flat, center=center)
    if dt is not None:
        vol = dt.Volume(DIMS, SPACING, (0.0, 0.0, 0.0), vol_np.astype(np.float64))
        spec = dt.DetectorSpec.for_volume(vol, H, W, (PITCH, PITCH))
        fixed = dt.render(vol, dt.PoseParameters.from_vector(TRUTH), spec).values
        _REF_STATE.update(vol=vol, spec=spec, fixed=fixed)
        return "reference", _ref_worker
    from oracle import oracle as O
    frame = O.pose_frame(np.asarray(TRUTH), center)
    _REF_STATE.update(fixed=O.render(flat, DIMS, SPACING, (0, 0, 0), frame, H, W, PITCH, PITCH))
    return "port", _port_worker


class CpuPool:
    """Fork pool of `procs` reference processes, created once."""

    def __init__(self, worker, procs):
        import multiprocessing as mp
        self.worker, self.procs = worker, procs
        self.pool = mp.get_context("fork").Pool(procs) if procs > 1 else None
        if self.pool is not None:  # import the reference in every worker before timing
            self.pool.map(_noop, range(procs), chunksize=1)

    def run(self, poses):
        t0 = time.perf_counter()
        if self.pool is None:
            res = [self.worker(p) for p in poses]
        else:
            res = self.pool.map(self.worker, list(poses), chunksize=1)
        return time.perf_counter() - t0, res

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()


def _noop(_):
    from oracle.oracle import reference_module
    reference_module()
    return 0


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(poses, budget_s):
    """The reference on this host: 1 process on 1 core, then os.cpu_count()
    processes (pose-sharded), on the GPU arm's own poses."""
    from paper_2208_12737_b200 import synthetic
    kind, worker = cpu_setup(synthetic.chest_phantom(DIMS))
    procs = os.cpu_count() or 1
    t1 = []
    t_start = time.perf_counter()
    i = 0
    while i < 2 or (time.perf_counter() - t_start < 0.2 * budget_s and i < 8):
        t1.append(worker(poses[i % len(poses)])[0])
        i += 1
    one_core = 1.0 / float(np.median(t1))
    pool = CpuPool(worker, procs)
    n = procs * max(1, int(0.8 * budget_s * one_core))
    n = min(n, procs * 64)
    wall, res = pool.run([poses[j % len(poses)] for j in range(n)])
    pool.close()
    return {
        "value": n / wall, "unit": "DRR/s", "cores": procs, "kind": kind,
        "one_core": {"value": one_core, "unit": "DRR/s", "cores": 1,
                     "sample": f"{len(t1)} poses, one at a time in this process"},
        "sample": f"{n} poses of the GPU arm's C2 batch (loss_and_gradient, neg-ZNCC, native "
                  f"backend, f64), pose-sharded over a {procs}-process fork pool created "
                  f"before timing; {wall:.1f} s wall; CPU {cpu_model()}"}


# ------------------------------------------------------------- GPU helpers
def make_timer(dev, flush):
    import torch
    stream = torch.cuda.current_stream(dev)

    def timed(fn, n, warm):
        out = []
        for i in range(n + warm):
            flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            if i >= warm:
                out.append(e0.elapsed_time(e1))
        return out
    return timed


def c5_volume(dev):
    """512^3 @ 0.703125 (sphere + 3x off-centre cube + noise), SURVEY 8(d) C5."""
    import torch
    n = 512
    c = (torch.arange(n, device=dev, dtype=torch.float64) + 0.5) * 0.703125
    mid, rad = n * 0.703125 / 2, 0.4 * n * 0.703125
    r2 = (c - mid)[:, None, None] ** 2 + (c - mid)[None, :, None] ** 2 + (c - mid)[None, None, :] ** 2
    frac = (torch.arange(n, device=dev, dtype=torch.float64) + 0.5) / n
    inb = (frac >= 0.25) & (frac <= 0.5)
    v5 = (r2 <= rad * rad).double() + 3.0 * (inb[:, None, None] & inb[None, :, None]
                                             & inb[None, None, :]).double()
    del r2
    gen = torch.Generator(device=dev).manual_seed(5)
    v5 = torch.clamp(v5 + 0.01 * torch.randn(v5.shape, device=dev, generator=gen,
                                             dtype=torch.float64) * (v5 > 0), min=0.0).float()
    return v5


def other_configs(sd, dev, timed, world, rank):
    """C1 / C3 / C4 / C5 of BASELINE.json on this node (parity-test cases in
    tests/test_gpu_configs.py; reported for context, not the headline).
    C4 and C5 are sharded over the ranks like the headline; C1 and C3 are
    single-pose configs and run on rank 0 only (N=1)."""
    import torch
    from paper_2208_12737_b200 import DeviceVolume, Detector, pose_frames, render_frames, synthetic
    from paper_2208_12737_b200.distributed import ShardedDRR, gather_rows, max_over_ranks
    out = {}
    # C4: C2 volume, 1024 narrow poses (seed 0), 256^2 @ 2.8125 mm, forward,
    # images collected on rank 0 through peer stores (and, for comparison, the
    # NCCL all-gather baseline of the same images)
    sd4 = sd.with_detector(Detector(256, 256, 2.8125))
    p4 = synthetic.sample_poses(TRUTH, synthetic.NARROW_HALF_WIDTHS, 1024, seed=0)
    p4_dev = torch.tensor(p4, device=dev)
    t = timed(lambda: sd4.render(p4_dev, copy=False), 5, 2)
    ms = max_over_ranks(float(np.median(t)), dev)
    out["C4"] = {"workload": f"C2 volume, 1024 narrow poses seed 0, 256x256 @2.8125 mm, forward, "
                             f"sharded over {world} GPU(s), images (268 MB) stored into rank 0's "
                             f"buffer by the forward kernels (peer memory)",
                 "ms_per_batch": ms, "drr_per_s": 1024 / (ms / 1e3)}
    if world > 1:
        lo, hi = sd4.shard(1024)
        fr = pose_frames(p4_dev[lo:hi], sd4.volume.center).detach()

        def nccl_gather():
            img = render_frames(sd4.volume, sd4.detector, fr)
            gather_rows(img, 1024)
        t = timed(nccl_gather, 5, 2)
        ms = max_over_ranks(float(np.median(t)), dev)
        out["C4"]["nccl_all_gather_baseline"] = {"ms_per_batch": ms, "drr_per_s": 1024 / (ms / 1e3)}
    sd4.close()
    if rank == 0 and world == 1:
        # C1: 128^3 sphere @ 1 mm, 100^2 @ 2.56 mm, one oblique pose, forward only
        v1 = DeviceVolume(synthetic.make_phantom("sphere", 128, 1.0), 1.0, device=dev)
        d1 = Detector(100, 100, 2.56)
        f1 = pose_frames(torch.tensor([[300.0, 0.4, 1.3, 0.1, 0.0, 0.0, 0.0]], device=dev),
                         v1.center).detach()
        t = timed(lambda: render_frames(v1, d1, f1), 20, 3)
        out["C1"] = {"workload": "128^3 sphere @1 mm, 100x100 @2.56 mm, 1 pose, forward",
                     "ms_per_drr": float(np.median(t))}
        # C3: 250-step registration (251 fwd+bwd iterations), one CUDA graph
        from paper_2208_12737_b200.registration import OptimizerConfig, RegistrationEngine
        with torch.no_grad():
            fixed = sd.render(np.asarray([TRUTH]))
        p0 = synthetic.sample_poses(TRUTH, synthetic.NARROW_HALF_WIDTHS, 1, seed=0)
        cfg = OptimizerConfig(converged_threshold=-1.1)
        eng = RegistrationEngine(sd.volume, sd.detector, fixed, 1, cfg)

        def reg_run():
            eng.reset(p0)
            eng.run(use_graph=True)
        reg_run()
        reg_ms = float(np.median(timed(reg_run, 3, 1)))
        # central finite differences reported alongside (north star):
        # default_fd_steps, float64 renders, boundary attribution (fd.fd_report)
        from paper_2208_12737_b200.fd import fd_report
        fd = {}
        eta2 = np.array([RHO, 0.4, 1.3, 0.1, 0.0, 0.0, 0.0])  # C2's single pose
        r2 = fd_report(sd.volume, sd.detector, eta2, fixed.double().cpu().numpy())
        fixed1 = render_frames(v1, d1, pose_frames(torch.tensor([[300.0, 0.45, 1.25, 0.1, 0.0, 0.0,
                                                                   0.0]], device=dev),
                                                   v1.center).detach(),
                               out_dtype=torch.float64)[0].cpu().numpy()
        r1 = fd_report(v1, d1, np.array([300.0, 0.4, 1.3, 0.1, 0.0, 0.0, 0.0]), fixed1)
        # at full scale (40000 rays x ~600 crossings) every default-step stencil
        # crosses some traversal-structure change; finer steps shrink the
        # kinked rays' share, so the FD error must shrink with the step
        fine = np.array([1e-5, 1e-7, 1e-7, 1e-7, 1e-5, 1e-5, 1e-5])
        r2f = fd_report(sd.volume, sd.detector, eta2, fixed.double().cpu().numpy(), steps=fine)
        for name, r in (("C2", r2), ("C2_fine_steps", r2f), ("C1", r1)):
            fd[name] = {k: r[k] for k in ("max_rel_kink_free", "n_kink_free", "boundary",
                                          "unexplained", "rel")}
        # ray by ray (fd.ray_fd_report): each ray's energy gradient vs its own
        # central FD, boundaries attributed per (ray, component)
        from paper_2208_12737_b200.fd import ray_fd_report
        for name, (vv, dd) in (("C2_rays", (sd.volume, sd.detector)), ("C1_rays", (v1, d1))):
            fd[name] = ray_fd_report(vv, dd, eta2)
        out["fd_check"] = {"method": "central FD, default_fd_steps (gradients.py:72-74), "
                                     "float64 renders; components whose stencil crosses a "
                                     "traversal-structure change (detect_fd_boundaries) are "
                                     "excluded; the reference's bar is rel < 1e-5. *_rays: the "
                                     "same per (ray, component) of the ray energies at C2's "
                                     "pose (fd.ray_fd_report)",
                           **fd}
        out["C3"] = {"workload": "slice-to-volume registration on C2: 250 momentum-GD steps "
                                 "(251 fwd+bwd iterations) of neg-ZNCC, whole loop one CUDA graph, "
                                 "3 launches per iteration (drr_register_step)",
                     "ms_total": reg_ms, "ms_per_step": reg_ms / (cfg.max_iters + 1),
                     "final_neg_zncc": eng.traces()[0].final_loss}
    # C5: 512^3 @ 0.703125, 1024^2 @ 0.703125, 64 poses fwd+bwd (loss_and_gradient
    # vs a fixed DRR at the truth pose), sharded, value + grad collected on rank 0
    v5 = c5_volume(dev) if rank == 0 else None
    sd5 = ShardedDRR(v5, 0.703125, RHO, 1024, 0.703125, device=dev)
    del v5
    fixed5 = sd5.render(np.asarray([TRUTH]))
    fx = [fixed5.cpu() if rank == 0 else None]
    if world > 1:
        import torch.distributed as dist
        dist.broadcast_object_list(fx, src=0)
    fixed5 = fx[0][0].to(dev)
    p5 = torch.tensor(synthetic.sample_poses(TRUTH, synthetic.NARROW_HALF_WIDTHS, 64, seed=0),
                      device=dev)
    t = timed(lambda: sd5.loss_and_gradient(p5, fixed5, copy=False), 3, 1)
    ms = max_over_ranks(float(np.median(t)), dev)
    out["C5"] = {"workload": f"512^3 @0.703125 sphere+3x cube+noise, 1024x1024 @0.703125, 64 poses "
                             f"fwd + neg-ZNCC + bwd, sharded over {world} GPU(s)",
                 "ms_per_batch": ms, "drr_per_s": 64 / (ms / 1e3)}
    sd5.close()
    del sd5
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------- main
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        return run_reference(args, world)

    import torch
    import torch.distributed as dist
    from paper_2208_12737_b200 import (backward_frames, backward_from_jac, count_steps,
                                       pose_frames, render_frames, render_frames_jac, synthetic)
    from paper_2208_12737_b200.distributed import ShardedDRR, max_over_ranks

    # DRR_BENCH_SHARED_GPU=1 (testing only) puts every rank on cuda:0 with the
    # gloo backend, so the multi-rank path can be exercised on a one-GPU box.
    shared = os.environ.get("DRR_BENCH_SHARED_GPU") == "1"
    dev = torch.device("cuda", 0 if shared else local)
    torch.cuda.set_device(dev)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    # --- volume: built on rank 0, broadcast once (NCCL over NVLink) -------
    vol_np = synthetic.chest_phantom(DIMS) if rank == 0 else None
    t0 = time.perf_counter()
    sd = ShardedDRR(vol_np, SPACING, RHO, H, PITCH, device=dev)
    torch.cuda.synchronize(dev)
    bcast_s = time.perf_counter() - t0
    del vol_np

    GB = args.batch
    poses = synthetic.sample_poses(TRUTH, synthetic.NARROW_HALF_WIDTHS, GB, seed=0)
    eta = torch.tensor(poses, device=dev)
    fixed = sd.render(np.asarray([TRUTH]))
    fx = [fixed.cpu() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(fx, src=0)
    fixed = fx[0][0].to(dev)
    lo, hi = sd.shard(GB)
    B = hi - lo

    def step():
        return sd.loss_and_gradient(eta, fixed, "neg_zncc", copy=False)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    timed = make_timer(dev, flush)

    # --- warmup + timed steps (device time, per-step events) -------------
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev.index) as clk:
        times = timed(step, args.steps, 0)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms_per_step = max_over_ranks(float(np.mean(times)), dev)
    value = GB / (ms_per_step / 1e3)
    # native launches per step on each rank (registration._Buffers picks the chain)
    mode = next(b.mode for k, b in sd._bufs.items() if k[0] == "lg")
    launches_per_step = 3 if mode == "jac" else 4
    chain = ("jac: pose_frames, forward_jac, loss_grad_jac" if mode == "jac" else
             "fused: pose_frames, forward_loss, image_loss, reduce_loss_grad")

    # --- e2e: public API, pinned host poses in, loss + grads back out ------
    h_eta = torch.tensor(poses).pin_memory()
    h_val = torch.empty(GB, dtype=torch.float64).pin_memory()
    h_grad = torch.empty((GB, 7), dtype=torch.float64).pin_memory()
    d_eta = torch.empty((GB, 7), dtype=torch.float64, device=dev)

    def e2e_step():
        d_eta[lo:hi].copy_(h_eta[lo:hi], non_blocking=True)  # this rank's poses
        r = sd.loss_and_gradient(d_eta, fixed, "neg_zncc", copy=False)
        if r is not None:
            h_val.copy_(r[0], non_blocking=True)
            h_grad.copy_(r[1], non_blocking=True)

    e2e_ms = max_over_ranks(float(np.mean(timed(e2e_step, args.steps, 3))), dev)
    e2e_value = GB / (e2e_ms / 1e3)
    if rank == 0:
        v_ref, g_ref = sd.loss_and_gradient(eta, fixed)
        torch.cuda.synchronize(dev)
        assert np.array_equal(h_val.numpy(), v_ref.cpu().numpy()), "e2e values differ"
        assert np.array_equal(h_grad.numpy(), g_ref.cpu().numpy()), "e2e gradients differ"
    else:
        sd.loss_and_gradient(eta, fixed)

    # --- the north-star nn.Module path (torch autograd), rank-local -------
    from paper_2208_12737_b200 import DRR
    from paper_2208_12737_b200.metrics import neg_zncc
    drr = DRR.from_device_volume(sd.volume, RHO, sd.detector, strict=False)
    rot0, tra0 = eta[lo:hi, 1:4], eta[lo:hi, 4:7]
    fixed_b = fixed.expand(B, H, W)

    def module_step():
        rot = rot0.detach().requires_grad_(True)
        tra = tra0.detach().requires_grad_(True)
        neg_zncc(drr(rot, tra), fixed_b).sum().backward()
    module_ms = float(np.mean(timed(module_step, max(10, args.steps // 5), 2)))

    # --- the dominant kernel against the roofline (this rank's shard) ----
    frames = pose_frames(eta[lo:hi], sd.volume.center).detach()
    # S: used voxel-steps of the reference's whole-volume walk;
    # S_walk: those the kernel takes (the occupied box; the rest add exact zeros)
    S = float(count_steps(sd.volume, sd.detector, frames, full=True).double().sum().item())
    S_walk = float(count_steps(sd.volume, sd.detector, frames).double().sum().item())
    g_img = torch.randn((B, H, W), device=dev, dtype=torch.float32)
    hold = {}

    def k_fj():
        hold["img"], hold["jac"] = render_frames_jac(sd.volume, sd.detector, frames)

    from paper_2208_12737_b200 import _lib as L
    lg_val = torch.empty(B, dtype=torch.float64, device=dev)
    lg_gf = torch.empty((B, 12), dtype=torch.float64, device=dev)

    def lgj(h):  # the step's tail: loss + pixel gradient + contraction (one launch)
        L.check(L.load().drr_loss_grad_jac(
            h["jac"].data_ptr(), h["img"].data_ptr(), fixed.data_ptr(), 0, 0, B,
            sd.detector.c, L.DRR_LOSS_NEG_ZNCC, lg_val.data_ptr(), None,
            lg_gf.data_ptr(), None, None, torch.cuda.current_stream(dev).cuda_stream))
    kfns = {"fj": k_fj,
            "bj": lambda: backward_from_jac(sd.detector, hold["jac"], g_img),
            "lgj": lambda: lgj(hold),
            "fwd": lambda: render_frames(sd.volume, sd.detector, frames),
            "rewalk": lambda: backward_frames(sd.volume, sd.detector, frames, g_img)}
    kt = {k: [] for k in kfns}
    for i in range(12):  # interleaved; the first two rounds are warm-up
        for name, fn in kfns.items():
            t = timed(fn, 1, 0)
            if i >= 2:
                kt[name].extend(t)
    kms = {k: float(np.mean(v)) for k, v in kt.items()}  # average launch duration, 10 launches
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    # SURVEY 8(d) algorithmic bytes of a forward walk: one fp32 gather per used
    # voxel-step + the fp32 image store; the stored Jacobian (48 B/pixel, an
    # artefact of this design) is reported beside it, not counted
    bytes_8d = 4.0 * S + 4.0 * B * H * W
    bytes_walk = 4.0 * S_walk + 4.0 * B * H * W  # what the kernel actually gathers + stores
    bytes_jac = 48.0 * B * H * W
    ncu = {}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)["k_forward_jac"]
        if tr.get("config") == "C2":
            per_pose = 1.0 / float(tr["poses"])  # capture scaled to this shard's pose count
            ncu = {"traffic": float(tr["traffic_bytes_per_launch"]) * per_pose * B,
                   "lts_bytes": (float(tr["lts_bytes_per_launch"]) * per_pose * B
                                 if "lts_bytes_per_launch" in tr else None),
                   "gather_sector_bytes": (float(tr["gather_sector_bytes_per_launch"]) * per_pose * B
                                           if "gather_sector_bytes_per_launch" in tr else None),
                   "l2_to_sm_bytes": (float(tr["l2_to_sm_bytes_per_launch"]) * per_pose * B
                                      if "l2_to_sm_bytes_per_launch" in tr else None),
                   "limiter": tr.get("limiter"), "limiter_frac": tr.get("limiter_frac"),
                   "capture": tr.get("source"), "capture_poses": tr.get("poses")}
    except (OSError, KeyError, ValueError):
        pass
    achieved = bytes_8d / (kms["fj"] / 1e3) / 1e9
    lts_gbs = (ncu["lts_bytes"] / (kms["fj"] / 1e3) / 1e9) if ncu.get("lts_bytes") else None
    # the north star's "ncu gather bandwidth": the 32-B sectors the gathers are
    # served at (L1 hits + misses) and the part of them that comes from L2
    gather_gbs = (ncu["gather_sector_bytes"] / (kms["fj"] / 1e3) / 1e9
                  if ncu.get("gather_sector_bytes") else None)
    l2sm_gbs = (ncu["l2_to_sm_bytes"] / (kms["fj"] / 1e3) / 1e9
                if ncu.get("l2_to_sm_bytes") else None)

    if world > 1:
        dist.barrier()
    other = None
    if not args.no_other_configs:
        other = other_configs(sd, dev, timed, world, rank)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(poses, args.cpu_seconds)

    if rank != 0:
        sd.close()
        dist.barrier()
        dist.destroy_process_group()
        return 0
    clocks = clk.summary()
    result = {
        "metric": METRIC,
        "value": value,
        "unit": "DRR/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (chest-shaped CT phantom, SURVEY 8(d)); random narrow poses",
        "config": {"workload": WORKLOAD, "global_batch": GB, "poses_per_gpu": B,
                   "detector": [H, W], "ct": list(DIMS), "parallelism": f"pose-shard x{world}",
                   "collect": "per-pose loss + 7-gradient stored into rank 0's buffers by the "
                              "kernels (peer memory over NVLink), inside the timed region",
                   "l2": "flushed (256 MiB write) between timed steps, outside the events",
                   "arithmetic": "f64 geometry, crossings and sums; the CT stored and gathered as fp32"},
        "e2e": {"value": e2e_value, "unit": "DRR/s",
                "h2d_bytes_per_step": int(GB * 7 * 8),
                "d2h_bytes_per_step": int(GB * 8 * 8),
                "api": "ShardedDRR.loss_and_gradient: pinned host poses -> device (each rank "
                       "its shard), loss + gradient read back to pinned host memory on rank 0"},
        "gpu_launches": launches_per_step * args.steps,
        "step_chain": chain,
        "module_path": {"api": "DRR nn.Module + metrics.neg_zncc + torch autograd (rank-local)",
                        "ms_per_step": module_ms, "value": B / (module_ms / 1e3)},
        "roofline": {"bound": "l1",
                     "roofline_of": "hbm",
                     "kernel": "k_forward_jac (the one CT walk per step: image + ray Jacobian)",
                     "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": ncu.get("traffic"),
                     "lts_gbs": lts_gbs,
                     "gather_bw": {"l1_sectors_gbs": gather_gbs,
                                   "l1_sectors_frac_of_hbm": (gather_gbs / hbm_peak
                                                              if gather_gbs else None),
                                   "l2_to_sm_gbs": l2sm_gbs,
                                   "l2_to_sm_frac_of_hbm": (l2sm_gbs / hbm_peak
                                                            if l2sm_gbs else None),
                                   "rule": "ncu l1tex__t_sectors_pipe_lsu_mem_global_op_ld x 32 B "
                                           "and l1tex__m_xbar2l1tex_read_bytes per launch (the "
                                           "capture, scaled per pose) / this run's launch time"},
                     "algorithmic_bytes_per_launch": bytes_8d,
                     "gathered_bytes_per_launch": bytes_walk,
                     "frac_gathered": bytes_walk / (kms["fj"] / 1e3) / 1e9 / hbm_peak,
                     "jacobian_store_bytes_per_launch": bytes_jac,
                     "bytes_rule": "SURVEY 8(d): 4 B per used voxel-step of the reference's "
                                   "whole-volume walk + 4 B per pixel; gathered_bytes counts the "
                                   "steps the kernel takes (its walk skips the volume's "
                                   "exactly-zero margins, bit-identically)",
                     "launch_ms": kms["fj"], "poses_per_launch": B,
                     "peak_source": "measured" if "hbm_gbs" in peaks else "fallback",
                     "limiter": ncu.get("limiter"), "limiter_frac": ncu.get("limiter_frac"),
                     "traffic_source": ncu.get("capture")},
        "kernels": {"forward_jac_ms": kms["fj"], "backward_jac_ms": kms["bj"],
                    "loss_grad_jac_ms": kms["lgj"],
                    "forward_only_ms": kms["fwd"], "rewalk_backward_ms": kms["rewalk"],
                    "voxel_steps_per_drr": S / B,
                    "walked_voxel_steps_per_drr": S_walk / B,
                    "voxel_steps_per_s_forward_jac": S / (kms["fj"] / 1e3),
                    "voxel_steps_per_s_forward_only": S / (kms["fwd"] / 1e3)},
        "ct_broadcast_s": bcast_s,
        "clocks": clocks,
    }
    if other is not None:
        result["other_configs"] = other
    if cpu is not None:
        result["cpu_baseline"] = cpu
    print(json.dumps(result))
    sd.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_reference(args, world):
    """--impl reference: the reference's own CPU path (oracle/_ref: drrtrace's
    loss_and_gradient, native Cython backend) on this host's cores, same
    metric and poses as the GPU arm; rank 0 only.  The fork pool is created
    once before the warm-up; each step is two poses per process, handed out
    one at a time (a step of one pose per process waits on its slowest pose:
    17.3 vs 22.4 DRR/s for the same pool on a long sample, rec4)."""
    from paper_2208_12737_b200 import synthetic
    kind, worker = cpu_setup(synthetic.chest_phantom(DIMS))
    procs = os.cpu_count() or 1
    poses = synthetic.sample_poses(TRUTH, synthetic.NARROW_HALF_WIDTHS, args.batch, seed=0)
    one = [worker(poses[i])[0] for i in range(3)]  # 1 process on 1 core first
    pool = CpuPool(worker, procs)
    times = []
    k = 0
    per_step = 2 * procs
    for i in range(max(args.warmup, 3) + args.steps):
        batch = [poses[(k + j) % len(poses)] for j in range(per_step)]
        k += per_step
        wall, _ = pool.run(batch)
        if i >= max(args.warmup, 3):
            times.append(wall)
    pool.close()
    ms = 1e3 * float(np.mean(times))
    value = per_step / (ms / 1e3)
    print(json.dumps({
        "impl": "reference",
        "metric": METRIC,
        "value": value, "unit": "DRR/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "global_batch": args.batch, "poses_per_step": per_step,
                   "parallelism": f"{procs} host processes"},
        "cpu_baseline": {"value": value, "unit": "DRR/s", "cores": procs, "kind": kind,
                         "one_core": {"value": 1.0 / float(np.median(one)), "unit": "DRR/s",
                                      "cores": 1, "sample": "3 poses, one at a time"},
                         "sample": f"{per_step} poses per step (two per process, dynamic) cycling through "
                                   f"the GPU arm's {args.batch}-pose batch, fork pool created "
                                   f"once before warm-up; CPU {cpu_model()}"},
        "e2e": {"value": value, "unit": "DRR/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))
    return 0


if __name__ == "__main__":
    sys.exit(main())
