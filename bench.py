#!/usr/bin/env python
"""Benchmark of the i-DEQ inference hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C3]

A *step* is one pass of the whole hot path over one batch: one inertial fixed-point
iteration (extrapolation, U-Net forward + input VJP, fidelity prox / step, per-image
residual) over the rank's images. Workload (N=1): BASELINE config C3, the "256^2 RGB
batch" the metric is quoted on: 32 images of 3x256x256 per GPU, U-Net-32, random
inpainting with the closed-form prox, bf16 tcgen05 convolutions. Under torchrun each
rank solves its own 32 images (weak scaling, no data-path collective for the
per-image stop rule). One JSON line is printed by rank 0.

Timing: W warm-up iterations, then EXACTLY K iterations in one ideq_solve call with
tol = 0, bracketed by a barrier and torch.cuda.synchronize on both sides, timed with
CUDA events on the solve stream; max over ranks. The per-iteration working set
(saved activations ~1 GB + iterate planes) is far larger than the 126 MB L2, so no
explicit flush is done (config.l2 says so).
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "image-iterations/s at 256² RGB batch; ms to fixed-point residual ≤1e-4"
UNIT = "image-iterations/s"


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML every 2 ms (the
    nvidia_ml_py binding), falling back to nvidia-smi every 100 ms."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index=0):
        self.index = index
        self.samples = []   # (sm_mhz, max_mhz, [4 bools])
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        n = self._nvml
        sm = n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM)
        mx = n.nvmlDeviceGetMaxClockInfo(self._h, n.NVML_CLOCK_SM)
        try:
            r = n.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            r = n.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        bits = [0x8, 0x40, 0x20, 0x4]   # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
        self.samples.append((float(sm), float(mx), [bool(r & b) for b in bits]))

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        parts = [p.strip() for p in out.stdout.strip().split(",")]
        if len(parts) >= 6 and parts[0].replace(".", "").isdigit():
            self.samples.append((float(parts[0]), float(parts[1]), [parts[2 + i].lower() == "active" for i in range(4)]))

    def _run(self):
        period = 0.002 if self._nvml else 0.1
        while not self._stop.is_set():
            try:
                self._sample_nvml() if self._nvml else self._sample_smi()
            except Exception:
                pass
            self._stop.wait(period)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"]}
        reasons = sorted({self.NAMES[i] for _, _, r in self.samples for i in range(4) if r[i]})
        return {"sm_mhz": statistics.median(x[0] for x in self.samples),
                "sm_max_mhz": max(x[1] for x in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi"}


def cpu_baseline(cfg, n_img=1, iters=3):
    """The fp64 oracle as it stands, on this host's cores: n_img images x iters iterations."""
    from oracle import solver as osolver
    from paper_2605_19705_b200 import synth
    prob = synth.make_problem(cfg, images=list(range(n_img)))
    net = osolver.make_net(cfg, prob["weights"])
    fids = osolver.make_fidelities(cfg, prob)
    t0 = time.perf_counter()
    osolver.solve(net, fids, prob["x0"], cfg["lam"], cfg["tau"], cfg["beta"], iters, 0.0, cfg["step"])
    dt = time.perf_counter() - t0
    return {"value": n_img * iters / dt, "unit": UNIT, "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
            "sample": f"{n_img} image x {iters} iterations of {cfg['name']} (fp64 numpy oracle, {dt:.1f} s)"}


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle on the host cores, on this arm's config and metric.
    Each step is one image-iteration of the same workload (a bounded sample)."""
    if rank != 0:
        return
    from oracle import solver as osolver
    from paper_2605_19705_b200 import synth
    prob = synth.make_problem(cfg, images=[0])
    net = osolver.make_net(cfg, prob["weights"])
    fids = osolver.make_fidelities(cfg, prob)
    x, xp = prob["x0"][0].astype(np.float64), prob["x0"][0].astype(np.float64)
    for _ in range(args.warmup):
        xn = osolver.ideq_step(x, xp, net, fids[0], cfg["lam"], cfg["tau"], cfg["beta"], cfg["step"])
        xp, x = x, xn
    t0 = time.perf_counter()
    for _ in range(args.steps):
        xn = osolver.ideq_step(x, xp, net, fids[0], cfg["lam"], cfg["tau"], cfg["beta"], cfg["step"])
        xp, x = x, xn
    dt = time.perf_counter() - t0
    v = args.steps / dt
    cores = len(os.sched_getaffinity(0))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config_dict(cfg, args.batch or (cfg["batch"] // 8 if args.config == "C5" else cfg["batch"]), world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"1 image-iteration of {cfg['name']} per step (fp64 numpy oracle)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config_dict(cfg, per_rank, world):
    opdesc = {"inpaint": f"{cfg['step']} inpainting (Bernoulli masks)",
              "blur": f"{cfg['step']} periodic blur {cfg.get('ksize')}x{cfg.get('ksize')} ({cfg.get('blur_impl', 'direct')})",
              "phase": f"{cfg.get('n_phase', 4)}-mask coded-diffraction phase retrieval (gradient)",
              "rician": "Rician denoising (gradient)", "mri": f"x{cfg.get('accel')} Cartesian MRI ({cfg['step']})"}[cfg["op"]]
    net = f"U-Net {'/'.join(map(str, cfg['widths']))}" if cfg["net"] == "unet4" else "tiny3"
    tag = cfg["name"].split()[0]
    return {"workload": f"{cfg['name']} (BASELINE config {tag}): {per_rank}x{cfg['C']}x{cfg['H']}x{cfg['W']} per GPU, "
                        f"{net}, {opdesc}, beta={cfg['beta']}",
            "global_batch": per_rank * world, "per_gpu_batch": per_rank, "H": cfg["H"], "W": cfg["W"],
            "C": cfg["C"], "net": f"unet4-{cfg['widths'][0]}" if cfg["net"] == "unet4" else "tiny3",
            "parallelism": f"dp{world}",
            "l2": "no flush: per-iteration working set (saved activations + iterate planes) >> 126 MB L2",
            "timed": "one ideq_solve of K iterations, tol=0 (no early stop)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--batch", type=int, default=0, help="images per GPU (default: the config's per-GPU batch)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--restart", type=float, default=0.0,
                    help="NEXT-1: adaptive restart with this B (Eq. 5, Alg. 1 semantics) in every timed solve")
    ap.add_argument("--averaging", action="store_true", help="NEXT-1: averaging (Alg. 1 steps 12-13) in the timed solves")
    ap.add_argument("--no-tol-run", action="store_true",
                    help="skip the ms-to-tolerance solve (the metric's second half: tol = 1e-4, per-image stop)")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference", "W >= 3 warm-up steps"

    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    from paper_2605_19705_b200 import configs
    cfg = configs.get(args.config)
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2605_19705_b200 import ideq, synth

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # per-GPU images: the config's batch, except C5 whose 512 images are sharded 64 per GPU at P = 8
    # (its weak-scaling unit); --batch overrides
    per = args.batch or (cfg["batch"] // 8 if args.config == "C5" else cfg["batch"])
    images = list(range(rank * per, (rank + 1) * per))
    prob = synth.make_problem(cfg, images=images)
    stream = torch.cuda.Stream()
    prec = cfg.get("precision", "bf16")   # C1 is an fp32 config (BASELINE), the others bf16
    s = ideq.Solver(cfg, prob["weights"], precision=prec, device=local, stream=stream, max_batch=per)
    s.set_operator(prob)
    y = torch.tensor(prob["y"]).cuda()
    x = torch.tensor(prob["x0"]).cuda()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world > 1:
            t = torch.tensor([v], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return v

    nx1 = dict(restart=1 if args.restart > 0 else 0, restart_B=args.restart, averaging=args.averaging)

    # ---- warm-up (also captures the CUDA graph of one iteration)
    s.solve(y, x, s.params(max_iter=args.warmup, tol=0.0, **nx1))
    x.copy_(torch.tensor(prob["x0"]))
    barrier()

    # ---- timed: exactly K iterations on device-resident inputs
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        stats, code, _ = s.solve(y, x, s.params(max_iter=args.steps, tol=0.0, **nx1))
        e1.record(stream)
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    assert (stats["iters"] == args.steps).all(), "timed solve did not run K iterations on every image"
    value = per * world * args.steps / (ms / 1000.0)

    # ---- e2e: same K iterations through ideq_solve_host (pinned host y/x, H2D + D2H inside)
    yh = torch.tensor(prob["y"]).pin_memory().numpy()
    xh = torch.tensor(prob["x0"]).pin_memory().numpy()
    # untimed warm-up of the host-buffer entry point (its staging buffers and the CUDA graph
    # captured for them), like the device-resident warm-up above
    s.solve_host(yh, xh.copy(), s.params(max_iter=args.warmup, tol=0.0, **nx1))
    barrier()
    t0 = time.perf_counter()
    s.solve_host(yh, xh, s.params(max_iter=args.steps, tol=0.0, **nx1))
    barrier()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e_v = per * world * args.steps / e2e_s

    # ---- roofline of the dominant kernel class (tcgen05 convolutions): CUDA events around
    #      every launch inside an eager (profiled) run of the same iterations
    kprof = min(args.steps, 10)
    x.copy_(torch.tensor(prob["x0"]))
    s.set_profiling(True)
    s.profile(reset=True)
    s.solve(y, x, s.params(max_iter=kprof, tol=0.0, **nx1))
    prof = s.profile(reset=True)
    s.set_profiling(False)
    peaks, peak_src = _peaks()
    tc = prof["conv_tc"]
    achieved = tc["flops"] / (tc["ms"] / 1000.0) / 1e12 if tc["ms"] > 0 else None
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    total_ms = sum(v["ms"] for v in prof.values())
    traffic = None
    tp = os.path.join(ROOT, "profiles", "conv_tc_traffic.json")
    if os.path.exists(tp) and args.config == "C3" and per == cfg["batch"]:  # captured on C3 only
        try:
            traffic = json.load(open(tp)).get("bytes_per_launch")
        except Exception:
            traffic = None
    if tc["ms"] == 0 and prof["conv_simt"]["ms"] > 0:  # FFMA path (C1 fp32): ALU roofline
        sm = prof["conv_simt"]
        ffma_peak = 148 * 128 * 2 * 1965e6 / 1e12   # derived: SMs x FP32 lanes x 2 x max SM clock
        roofline = {"bound": "alu", "achieved": sm["flops"] / (sm["ms"] / 1000.0) / 1e12, "peak": ffma_peak,
                    "unit": "TFLOP/s", "frac": sm["flops"] / (sm["ms"] / 1000.0) / 1e12 / ffma_peak, "traffic": None,
                    "kernel": "conv_simt_kernel (all FFMA conv launches of a step)",
                    "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 FLOP x 1965 MHz",
                    "share_of_step": sm["ms"] / total_ms if total_ms else None,
                    "per_class_ms_per_step": {k: v["ms"] / kprof for k, v in prof.items()},
                    "algorithmic_flops_per_step": sm["flops"] / kprof}
    else:
      roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "kernel": "conv_tc_kernel (all tcgen05 conv launches of a step)",
                "peak_source": f"{peak_src} bf16_tflops_sustained (kernel timed inside the step)",
                "share_of_step": tc["ms"] / total_ms if total_ms else None,
                "per_class_ms_per_step": {k: v["ms"] / kprof for k, v in prof.items()},
                "algorithmic_flops_per_step": tc["flops"] / kprof,
                # algorithmic HBM bytes per launch (each activation read / written once, weights
                # once) beside the ncu-measured `traffic` of the same launches
                "algorithmic_bytes_per_launch": (tc["bytes"] / tc["launches"]) if tc["launches"] else None}

    # ---- ms to tolerance (tol = 1e-4, per-image stop)
    tol_info = None
    if not args.no_tol_run and not args.averaging:  # averaging needs a fixed iteration count (reading R5)
        x.copy_(torch.tensor(prob["x0"]))
        barrier()
        e0.record(stream)
        st2, _, _ = s.solve(y, x, s.params(max_iter=cfg["max_iter"], tol=1e-4, **nx1))
        e1.record(stream)
        barrier()
        tol_info = {"ms": max_over_ranks(e0.elapsed_time(e1)), "tol": 1e-4,
                    "iters_max": int(st2["iters"].max()), "iters_mean": float(st2["iters"].mean()),
                    "converged": int((st2["status"] == 0).sum()), "images": per}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if prec == "fp32" else "bf16", "data": "synthetic (seeded piecewise-smooth images, random-init "
            "U-Net weights" + {"inpaint": "; stands in for the paper's BSDS500 inpainting split)",
                               "mri": "; stand-in phantoms for the paper's fastMRI knee data)"}.get(cfg["op"], ")"),
            "config": dict(_config_dict(cfg, per, world), **({"restart_B": args.restart} if args.restart > 0 else {}),
                           **({"averaging": True} if args.averaging else {})),
            "e2e": {"value": e2e_v, "unit": UNIT, "h2d_bytes_per_step": (yh.nbytes + xh.nbytes) / args.steps,
                    "d2h_bytes_per_step": xh.nbytes / args.steps,
                    "note": "one ideq_solve_host call of K iterations: H2D of y and x0, D2H of x-hat inside"},
            "gpu_launches": s.launches_per_iteration() * args.steps + 4,
            "roofline": roofline, "clocks": clk.summary()}
    if tol_info:
        line["ms_to_tolerance"] = tol_info
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
