"""Helpers for the -m gpu tests (device tensors, layout conversion, metrics)."""
import numpy as np


def torch_cuda():
    import pytest
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float64 (what the GPU sees)."""
    import torch
    return torch.tensor(np.asarray(a, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def nhwc_dev(x_nchw: np.ndarray, dtype: str):
    import torch
    t = torch.tensor(np.ascontiguousarray(np.asarray(x_nchw, dtype=np.float32).transpose(0, 2, 3, 1)))
    t = t.to(torch.bfloat16 if dtype == "bf16" else torch.float32)
    return t.cuda().contiguous()


def from_nhwc_dev(t) -> np.ndarray:
    import torch
    return t.to(torch.float32).cpu().numpy().transpose(0, 3, 1, 2).astype(np.float64)


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def psnr(x, ref, peak=1.0) -> float:
    """10 log10(peak^2 / MSE) over all entries of one image (reading Q21)."""
    mse = float(np.mean((np.asarray(x, np.float64) - np.asarray(ref, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(peak * peak / mse)
