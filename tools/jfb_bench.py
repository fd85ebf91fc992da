"""Measure the JFB training gradient through the C ABI `ideq_jfb_grad`.

One call = one JFB gradient over a batch at x_hat: grad g and U (the solver's network), the
residual, the two-stream forward with tape, the reverse with weight gradients, the D2H of dtheta.
Timed with CUDA events around the synchronous call, after warm-up (the call's tape cudaMallocs
are inside the timed region: this is the user-visible call latency). Algorithmic FLOPs: F = one
forward of the U-Net convolutions on the batch; the call issues ~8F (grad g = forward + VJP = 2F,
two-stream forward 2F, two-stream adjoints 2F, two-stream weight gradients 2F). In the fp32 mode
the U-Net convolutions of grad g and of the two-stream passes run on tcgen05 (3xTF32) and the weight
gradients on FFMA; `frac` is quoted against the derived FFMA peak (148 SMs x 128 lanes x 2 FLOP x
1965 MHz = 74.4 TFLOP/s) for comparability with the round-1 lines, where every pass was FFMA.
The oracle (oracle/jfb.py, fp64, 1 image) is timed beside it on the host.

usage: python tools/jfb_bench.py [--config C3] [--batch 4] [--steps 5] [--warmup 2]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_19705_b200 import configs, synth  # noqa: E402

FFMA_PEAK = 148 * 128 * 2 * 1965e6 / 1e12


def unet_forward_flops(cfg, N):
    H, W, C = cfg["H"], cfg["W"], cfg["C"]
    w = cfg["widths"]
    if cfg["net"] == "tiny3":
        return 2.0 * N * H * W * 9 * (C * w[0] + w[0] * w[0] + w[0] * C)
    R = cfg.get("res_blocks", 2)
    f = 2 * 2.0 * N * H * W * 9 * C * w[0]                           # head + tail
    for l in range(4):
        hw = (H >> l) * (W >> l)
        nrb = R * (2 if l < 3 else 1)                                  # encoder + decoder blocks
        f += nrb * 2 * 2.0 * N * hw * 9 * w[l] * w[l]
        if l < 3:
            f += 2 * 2.0 * N * ((H >> (l + 1)) * (W >> (l + 1))) * 4 * w[l] * w[l + 1]   # down + up
    return f


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--no-oracle", action="store_true")
    a = ap.parse_args()
    import torch
    from paper_2605_19705_b200 import ideq
    cfg = configs.get(a.config, batch=a.batch, init_scale=0.3)
    prob = synth.make_problem(cfg)
    s = ideq.Solver(cfg, prob["weights"], precision="fp32", max_batch=cfg["batch"])
    s.set_operator(prob)
    xs = prob["x_true"].astype(np.float32)
    x_hat = (0.9 * xs + 0.05).astype(np.float32)
    dev = lambda t: torch.tensor(np.ascontiguousarray(t, dtype=np.float32)).cuda()
    y, xh, xst = dev(prob["y"]), dev(x_hat), dev(xs)
    p = s.params()
    for _ in range(a.warmup):
        s.jfb_grad(y, xh, xst, p)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        loss, dth, dlam, dtau, _ = s.jfb_grad(y, xh, xst, p)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    F = unet_forward_flops(cfg, cfg["batch"])
    out = {"what": "ideq_jfb_grad", "config": a.config, "batch": cfg["batch"], "H": cfg["H"], "W": cfg["W"],
           "widths": list(cfg["widths"]), "step": cfg["step"], "ms_per_call": ms,
           "images_per_s": cfg["batch"] / (ms / 1e3), "algorithmic_tflops": 8 * F / (ms / 1e3) / 1e12,
           "ffma_peak_tflops_derived": FFMA_PEAK, "frac": 8 * F / (ms / 1e3) / 1e12 / FFMA_PEAK,
           "loss": loss, "dlam": dlam, "dtau": dtau, "dtheta_norm": float(np.linalg.norm(dth))}
    if not a.no_oracle:
        from oracle import jfb
        from oracle import solver as osolver
        net = osolver.make_net(cfg, prob["weights"])
        fid = osolver.make_fidelities(cfg, prob)[0]
        t0 = time.perf_counter()
        jfb.jfb_grads(net, fid, x_hat[0].astype(np.float64), xs[0].astype(np.float64), cfg["lam"], cfg["tau"],
                      cfg["step"])
        dt = time.perf_counter() - t0
        out["oracle_s_per_image"] = dt
        out["oracle_sample"] = "1 image, fp64, oracle/jfb.py as it stands"
        out["speedup_vs_oracle"] = (cfg["batch"] / (ms / 1e3)) * dt
    print(json.dumps(out))


if __name__ == "__main__":
    main()
