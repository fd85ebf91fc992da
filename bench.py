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
            "cpu_model": _cpu_model(),
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
            "config": dict(_config_dict(cfg, args.batch or (cfg["batch"] // world if args.config == "C5" else cfg["batch"]),
                                        world), timed_images_per_step=1,
                           timed="one image-iteration of the same workload per step (a bounded sample of the batch)"),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": _cpu_model(),
                             "sample": f"1 image-iteration of {cfg['name']} per step (fp64 numpy oracle)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _relaunch_under_torchrun(args):
    """`bench.py --gpus N` without a torchrun environment: start N ranks on this node (one process
    per GPU) through torch.distributed.run, with the same arguments; rank 0 prints the line."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


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


def _tiny_roofline(cfg, per, step_ms):
    """C1's whole-solve kernel (one P-SM cluster per image, P = 16 when H allows, else 8): ALU
    roofline of the algorithmic FLOPs (network forward + input VJP, 2 FLOP / MAC, and the blur A z,
    A^T r) against the chip's derived FFMA peak and against the P SMs one image's cluster can use."""
    w, C, HW, ks = cfg["widths"][0], cfg["C"], cfg["H"] * cfg["W"], cfg["ksize"]
    macs = 9 * (C * w + w * w + w * C) * HW * 2 + 2 * ks * ks * HW * C
    flops = 2.0 * macs * per
    ach = flops / (step_ms / 1000.0) / 1e12
    chip = 148 * 128 * 2 * 1965e6 / 1e12
    P = 16 if cfg["H"] % 16 == 0 and (cfg["H"] // 16) % 2 == 0 else 8   # tiny_solve.cu ts_cluster
    cluster = P * 128 * 2 * 1965e6 / 1e12 * per
    return {"bound": "alu", "achieved": ach, "peak": chip, "unit": "TFLOP/s", "frac": ach / chip, "traffic": None,
            "kernel": f"tiny_solve_kernel (the whole solve in one launch, one {P}-CTA cluster per image)",
            "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 FLOP x 1965 MHz",
            "frac_of_cluster_sms": ach / cluster, "us_per_iteration": step_ms * 1000.0,
            "algorithmic_flops_per_step": flops, "launches_per_solve": 1}


def _class_roofline(s, cfg, prec, per, args, ms, clk, peaks, peak_src):
    cls = "conv_tc" if prec == "bf16" or cfg["net"] == "unet4" else "conv_simt"
    reps = 20
    kt = s.time_class(cls, reps)
    st_t = s.time_class("step", reps)
    ht_t = s.time_class("headtail", reps)
    clocks = clk.summary()
    # the class's time inside the device-timed step: its share of the bracketed iteration (event
    # nodes at class boundaries of the replayed graph) times the step's own duration
    step_ms = ms / args.steps
    conv_ms = kt["share"] * step_ms
    burst = bool(clocks.get("sm_mhz") and clocks.get("sm_max_mhz") and ms < 1000.0
                 and clocks["sm_mhz"] >= 0.97 * clocks["sm_max_mhz"])
    if cls == "conv_simt":   # FFMA convolutions (C1's tiny net): ALU roofline
        ffma_peak = 148 * 128 * 2 * 1965e6 / 1e12   # derived: SMs x FP32 lanes x 2 x max SM clock
        ach = kt["flops"] / (conv_ms / 1000.0) / 1e12
        roofline = {"bound": "alu", "achieved": ach, "peak": ffma_peak, "unit": "TFLOP/s", "frac": ach / ffma_peak,
                    "traffic": None, "kernel": "conv_simt_kernel (all FFMA conv launches of a step)",
                    "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 FLOP x 1965 MHz"}
    else:
        # tensor peak of the path's own dtype: bf16 measured; 3xTF32 = measured bf16 x (TF32/bf16
        # nominal ratio 1/2) / 3 MMAs per product
        scale = 1.0 if prec == "bf16" else 0.5 / 3.0
        pk_b = peaks.get("bf16_tflops") * scale
        pk_s = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")) * scale
        peak = pk_b if burst else pk_s
        ach = kt["flops"] / (conv_ms / 1000.0) / 1e12
        traffic = None
        tp = os.path.join(ROOT, "profiles", "conv_tc_traffic.json")
        if os.path.exists(tp) and args.config == "C3" and per == cfg["batch"] and prec == "bf16":
            try:
                traffic = json.load(open(tp)).get("bytes_per_launch")
            except Exception:
                traffic = None
        roofline = {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                    "traffic": traffic,
                    "kernel": "conv_tc_kernel (all tcgen05 conv launches of a step)" + ("" if prec == "bf16" else
                              ", 3xTF32 (kind::tf32, 3 MMAs per product)"),
                    "peak_source": f"{peak_src} {'bf16_tflops (burst: sub-second region at max clock)' if burst else 'bf16_tflops_sustained'}"
                                   + ("" if prec == "bf16" else " x 1/2 (TF32 nominal) / 3 (3xTF32)"),
                    "frac_burst": ach / pk_b, "frac_sustained": ach / pk_s}
    roofline.update({
        "timing": f"ideq_time_class: event-record nodes at the class boundaries of one captured iteration, {reps} replays",
        "ms_per_step": conv_ms, "share_of_step": kt["share"],
        "class_ms_in_replay": kt["ms"], "replayed_iteration_ms": kt["iter_ms"],
        "algorithmic_flops_per_step": kt["flops"], "algorithmic_bytes_per_step": kt["bytes"],
        "launches_per_step": s.launches_per_iteration(),
        "other_classes_ms_per_step": {"step": st_t["ms"], "headtail": ht_t["ms"]},
        "step_kernel": {"bound": "hbm", "algorithmic_bytes_per_step": st_t["bytes"], "ms": st_t["ms"],
                        "achieved_gbs": st_t["bytes"] / (st_t["ms"] / 1000.0) / 1e9,
                        "frac": st_t["bytes"] / (st_t["ms"] / 1000.0) / 1e9 / peaks["hbm_gbs"],
                        "peak_gbs": peaks["hbm_gbs"],
                        "timing": "event nodes around the update's launches in the replayed iteration"},
    })
    return roofline


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--batch", type=int, default=0, help="images per GPU (default: the config's per-GPU batch)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--precision", default=None, choices=["bf16", "fp32"],
                    help="override the config's precision (fp32 = the 3xTF32 tensor-core parity mode)")
    ap.add_argument("--restart", type=float, default=0.0,
                    help="NEXT-1: adaptive restart with this B (Eq. 5, Alg. 1 semantics) in every timed solve")
    ap.add_argument("--averaging", action="store_true", help="NEXT-1: averaging (Alg. 1 steps 12-13) in the timed solves")
    ap.add_argument("--no-tol-run", action="store_true",
                    help="skip the ms-to-tolerance solve (the metric's second half: tol = 1e-4, per-image stop)")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference", "W >= 3 warm-up steps"

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch_under_torchrun(args))
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"
    from paper_2605_19705_b200 import configs
    cfg = configs.get(args.config)
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2605_19705_b200 import dist as dist_util
    from paper_2605_19705_b200 import ideq, synth

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # per-GPU images: the config's batch on every rank (weak scaling: the per-GPU work is fixed),
    # except C5 whose 512 images are sharded over the ranks (the largest batch, BASELINE C5);
    # --batch overrides
    if args.config == "C5" and not args.batch:
        shard = dist_util.shard(cfg["batch"], world, rank)
        images, scaling = list(shard), "strong"
    else:
        per0 = args.batch or cfg["batch"]
        images, scaling = list(range(rank * per0, (rank + 1) * per0)), "weak"
    per = len(images)
    prob = synth.make_problem(cfg, images=images)
    stream = torch.cuda.Stream()
    prec = args.precision or cfg.get("precision", "bf16")   # C1 is an fp32 config (BASELINE), the others bf16
    # NCCL communicator for the GLOBAL_MAX stop rule (C5): rank 0 draws the id, torch.distributed
    # broadcasts it; per-image configs need no collective
    nccl_id = None
    if world > 1 and cfg["stop_rule"] == "global_max":
        nccl_id = dist_util.broadcast_nccl_id()
    s = ideq.Solver(cfg, prob["weights"], precision=prec, device=local, stream=stream, max_batch=per,
                    rank=rank, world=world, nccl_id=nccl_id)
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
    value = (cfg["batch"] if scaling == "strong" else per * world) * args.steps / (ms / 1000.0)

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
    e2e_v = (cfg["batch"] if scaling == "strong" else per * world) * args.steps / e2e_s

    # ---- roofline of the dominant kernel class: its launches of one iteration, in the iteration's
    #      order and launch configuration, captured into one CUDA graph and replayed back to back
    #      (ideq_time_class: CUDA events on the solve stream); its share of the device-timed step
    peaks, peak_src = _peaks()
    if s.launches_per_iteration() == 0:
        roofline = _tiny_roofline(cfg, per, ms / args.steps)
    else:
        roofline = _class_roofline(s, cfg, prec, per, args, ms, clk, peaks, peak_src)
    clocks = clk.summary()

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
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32" if prec == "fp32" else "bf16", "data": "synthetic (seeded piecewise-smooth images, random-init "
            "U-Net weights" + {"inpaint": "; stands in for the paper's BSDS500 inpainting split)",
                               "mri": "; stand-in phantoms for the paper's fastMRI knee data)"}.get(cfg["op"], ")"),
            "config": dict(_config_dict(cfg, per, world), **({"restart_B": args.restart} if args.restart > 0 else {}),
                           **({"averaging": True} if args.averaging else {})),
            "e2e": {"value": e2e_v, "unit": UNIT, "h2d_bytes_per_step": (yh.nbytes + xh.nbytes) / args.steps,
                    "d2h_bytes_per_step": xh.nbytes / args.steps,
                    "note": "one ideq_solve_host call of K iterations: H2D of y and x0, D2H of x-hat inside"},
            "gpu_launches": (s.launches_per_iteration() * args.steps + 4) if s.launches_per_iteration() else 1,
            "roofline": roofline, "clocks": clocks, "plan": s.plan()}
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
