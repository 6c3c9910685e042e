#!/usr/bin/env python
"""FFST benchmark: forward + inverse (adjoint) over a batch of synthetic images.

One step = one pass of the whole hot path (image spectrum, forward transform to
the complex coefficient cube, inverse transform back to the images) over one
batch, i.e. every row of SURVEY.md 8(a).  Default workload: BASELINE.json
configs[1] (256x256 float32, batch 16).  Prints ONE JSON line (rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

N > 1 (launched by torch.distributed.run): the eta shearlet planes are sharded
(plane i on rank i mod N); rank 0 broadcasts the images (NCCL), every rank runs
its planes, the partial images are reduced to rank 0 (NCCL).  Total work is
fixed as N grows ("strong").  --impl reference times the float64 oracle (the
paper-faithful CPU program) on host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "FFST forward+inverse images/s and coeff GB/s at 1/2/4/8 B200; % HBM peak"
L2_FLUSH_BYTES = 512 << 20


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------ oracle arm

def oracle_images_per_s(cfg, budget_s: float, max_images: int):
    """The float64 oracle (as it stands) on host cores: forward + inverse of images of
    the config one by one (spectra built once and reused, as the paper caches them,
    P:L2207) until `budget_s` of CPU work.  Returns (images/s, images, seconds)."""
    import oracle as O
    psi = O.shearlet_spectra(cfg.n)
    done, dt = 0, 0.0
    while done < max_images:
        x = synth.make_image(cfg, done % cfg.batch).astype(np.float32 if cfg.dtype == "f32" else np.float64)
        t0 = time.perf_counter()
        c = O.forward(x.astype(np.float64), psi=psi)
        O.inverse(c, psi=psi)
        dt += time.perf_counter() - t0
        done += 1
        if dt >= budget_s:
            break
    return done / dt, done, dt


def oracle_cores():
    # numpy.fft (pocketfft) and the vectorised window code run single-threaded
    return 1


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    workload = f"config{cfg.cid}"
    per_step = []
    imgs = 0
    for s in range(args.warmup + args.steps):
        x = synth.make_image(cfg, s % max(cfg.batch, 1))
        import oracle as O
        if s == 0:
            psi = O.shearlet_spectra(cfg.n)
        t0 = time.perf_counter()
        c = O.forward(x.astype(np.float32 if cfg.dtype == "f32" else np.float64).astype(np.float64), psi=psi)
        O.inverse(c, psi=psi)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            per_step.append(dt)
            imgs += 1
    total = sum(per_step)
    value = imgs / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * total / len(per_step), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload, "n": cfg.n, "batch_per_step": 1, "config_batch": cfg.batch,
                   "label": cfg.label},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": oracle_cores(), "kind": "oracle",
                         "sample": f"1 image of {workload} per step (forward+inverse, float64 numpy oracle, "
                                   f"spectra cached), {imgs} timed steps"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ GPU arm

def run_gpu(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_1202_1773_b200 as F

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    dtype = torch.float32 if cfg.dtype == "f32" else torch.float64
    rsz = 4 if dtype == torch.float32 else 8
    B, N = cfg.batch, cfg.n

    plan = F.Plan(N, B, dtype, device=dev, shard_rank=rank, shard_count=world)
    eta, eta_l = plan.eta, plan.eta_local
    x_host = torch.from_numpy(synth.make_batch(cfg.cid)).to(dtype)
    x = x_host.to(dev) if rank == 0 else torch.empty(B, N, N, dtype=dtype, device=dev)
    cube = plan.empty_coeffs()
    rec = plan.empty_images()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    if world > 1:
        from paper_1202_1773_b200.dist import ShardedTransform
        sharded = ShardedTransform(plan)

        def step():
            dist.broadcast(x, src=0)                       # images in (NCCL)
            plan.forward(x, out=cube)                      # local planes
            sharded.inverse(cube, out=rec)                 # partial image, NCCL reduce to rank 0
    else:
        def step():
            plan.forward(x, out=cube)
            plan.inverse(cube, out=rec)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    # quick correctness guard on the measured configuration (round trip, rank 0)
    if rank == 0:
        rt_err = float((rec - x).abs().max() / x.abs().max())
    else:
        rt_err = None

    plan.set_timing(True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    fwd_main, inv_main = [], []
    launches = (0, 0)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()                                  # L2 flush between timed steps (untimed)
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
            torch.cuda.synchronize(dev)
            (tf, ti, _, _), launches = plan.phase_times()
            fwd_main.append(tf)
            inv_main.append(ti)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
    plan.set_timing(False)
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_step = total_ms / args.steps
    images_s = B * args.steps / (total_ms / 1000.0)
    cube_bytes = B * eta * N * N * 2 * rsz                 # whole-job cube, written once + read once
    coeff_gbs = 2 * cube_bytes / (ms_step / 1000.0) / 1e9
    algo_bytes = B * N * N * (2 * rsz + 2 * eta * 2 * rsz)  # (8 + 16 eta) N^2 per image in f32
    peak, peak_src = peaks()
    hbm_frac_step = algo_bytes / world / (ms_step / 1000.0) / 1e9 / peak

    # dominant kernel roofline: the persistent forward / inverse kernels (per-rank cube stream)
    fm, im = float(np.mean(fwd_main)), float(np.mean(inv_main))
    local_cube = B * eta_l * N * N * 2 * rsz
    dom_name, dom_ms = ("fwd_main", fm) if fm >= im else ("inv_main", im)
    achieved = local_cube / (dom_ms / 1000.0) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as fh:
                traffic = json.load(fh).get(f"config{cfg.cid}", {}).get(dom_name)
        except Exception:
            traffic = None
    clocks = clk.summary()

    # end to end through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if world == 1:
        x_pin = x_host.pin_memory()
        out_pin = torch.empty(B, N, N, dtype=dtype).pin_memory()
        for _ in range(2):
            plan.forward_host(x_pin, out=cube)
            plan.inverse_host(cube, out_pin)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_ms = 0.0
        for _ in range(args.steps):
            flush.zero_()
            e0.record(stream)
            plan.forward_host(x_pin, out=cube)
            plan.inverse_host(cube, out_pin)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            e_ms += e0.elapsed_time(e1)
        e2e = {"value": B * args.steps / (e_ms / 1000.0), "unit": "images/s",
               "h2d_bytes_per_step": B * N * N * rsz, "d2h_bytes_per_step": B * N * N * rsz}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, n_img, secs = oracle_images_per_s(cfg, budget_s=args.cpu_budget, max_images=max(cfg.batch, 4) * 4)
        cpu = {"value": v, "unit": "images/s", "cores": oracle_cores(), "kind": "oracle",
               "sample": f"{n_img} images of config{cfg.cid} ({N}x{N}), forward+inverse each, float64 numpy "
                         f"oracle, spectra built once (cached), {secs:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": images_s, "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if dtype == torch.float32 else "f64", "data": "synthetic",
            "config": {"workload": f"config{cfg.cid}", "label": cfg.label, "n": N, "global_batch": B,
                       "j0": plan.j0, "eta": eta, "parallelism": f"eta-shard{world}" if world > 1 else "single",
                       "l2": "flushed between timed steps (512 MiB write, untimed)"},
            "coeff_gbs": coeff_gbs,
            "hbm_frac_step": hbm_frac_step,
            "algorithmic_bytes_per_step": algo_bytes,
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "peak_source": peak_src,
                         "bytes_per_launch": local_cube,
                         "kernel_ms": {"fwd_main": fm, "inv_main": im}},
            "cpu_baseline": cpu,
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": (launches[0] + launches[1]) * args.steps,
            "roundtrip_max_rel_err": rt_err,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, help="BASELINE.json configs[C-1] (1..5)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = synth.config(args.config)
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_gpu(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
