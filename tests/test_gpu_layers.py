"""Per-layer parity of the network convolutions (tcgen05 and FFMA paths) against the
oracle's layer definitions, through include/ideq_debug.h."""
import numpy as np
import pytest

from oracle import nets
from tests.gpu_util import bf16_round, from_nhwc_dev, nhwc_dev, rel_l2, torch_cuda

pytestmark = pytest.mark.gpu

# kind -> (oracle function, weight shape builder, input-channel index, output-channel index,
#          input spatial (given the test's fine H, W), output spatial)
KINDS = {
    0: (nets.conv3x3, lambda a, b: (b, a, 3, 3)),          # in a -> out b, W [co=b][ci=a]
    1: (nets.conv3x3_T, lambda a, b: (a, b, 3, 3)),        # in a = co -> out b = ci, W [co=a][ci=b]
    2: (nets.down2x2, lambda a, b: (b, a, 2, 2)),          # fine a -> coarse b
    3: (nets.down2x2_T, lambda a, b: (a, b, 2, 2)),        # coarse a (=co) -> fine b (=ci)
    4: (nets.up2x2, lambda a, b: (a, b, 2, 2)),            # coarse a (=ci) -> fine b (=co), Wu [ci][co]
    5: (nets.up2x2_T, lambda a, b: (b, a, 2, 2)),          # fine a (=co) -> coarse b (=ci), Wu [ci=b][co=a]
}


def _spatial(kind, H, W):
    """(input H, W) for the kind given a fine-grid H x W."""
    return (H // 2, W // 2) if kind in (3, 4) else (H, W)


def _epi_ref(acc, epi, aux):
    if epi == 1:
        return nets.softplus(acc)
    if epi == 2:
        return acc + aux
    if epi == 3:
        return acc * (-np.expm1(-aux))
    return acc


def assert_elementwise(got, ref, prec):
    """Element-wise bound (catches errors confined to a few tile edges that a whole-tensor norm
    would average away): bf16 outputs carry one rounding of 2^-9 relative to each element, so
    max|got - ref| <= 2^-8 max|ref|; fp32 accumulation over <= 9 x 256 products stays far below
    1e-5 max|ref|."""
    bound = (2.0 ** -8 if prec == "bf16" else 1e-5) * np.abs(ref).max()
    err = np.abs(got - ref)
    assert err.max() <= bound, (prec, float(err.max()), float(bound), np.unravel_index(err.argmax(), err.shape))


CASES = []
for kind in range(6):
    pairs = [(32, 32), (64, 128)] + ([(64, 64)] if kind in (0, 1) else [])   # (64,64): resident-weight halo path
    for cin, cout in pairs:
        for (H, W) in [(20, 40), (8, 272)]:
            if kind in (2, 3, 4, 5) and (H % 2 or W % 2):
                continue
            for epi in (0, 1, 2, 3):
                CASES.append((kind, cin, cout, H, W, epi))


@pytest.mark.parametrize("path", ["fp32", "fp32-tc", "bf16-simt", "bf16-tc"])
@pytest.mark.parametrize("kind,cin,cout,H,W,epi", CASES)
def test_layer_vs_oracle(path, kind, cin, cout, H, W, epi):
    """Paths: fp32 FFMA (the JFB gradient's convolutions), fp32 on tcgen05 as 3xTF32 (the parity
    mode's network), bf16 FFMA, bf16 tcgen05 (the headline)."""
    torch = torch_cuda()
    from paper_2605_19705_b200 import ideq
    prec = "fp32" if path.startswith("fp32") else "bf16"
    use_tc = path.endswith("-tc")
    rng = np.random.default_rng(hash((kind, cin, cout, H, W, epi)) % (2 ** 32))
    fn, wshape = KINDS[kind]
    w = rng.standard_normal(wshape(cin, cout)) * np.sqrt(1.0 / (cin * 4))
    Hin, Win = _spatial(kind, H, W)
    N = 2
    x = rng.standard_normal((N, cin, Hin, Win))
    w32 = w.astype(np.float32)
    if prec == "bf16":
        xr, wr = bf16_round(x), bf16_round(w32)
    else:
        xr, wr = x.astype(np.float32).astype(np.float64), w32.astype(np.float64)
    ref_acc = np.stack([fn(xr[n], wr) for n in range(N)])
    aux = None
    auxr = None
    if epi in (2, 3):
        aux = rng.uniform(0.05, 2.0, ref_acc.shape) if epi == 3 else rng.standard_normal(ref_acc.shape)
        auxr = bf16_round(aux) if prec == "bf16" else aux.astype(np.float32).astype(np.float64)
    ref = _epi_ref(ref_acc, epi, auxr)
    xin = nhwc_dev(x, prec)
    out = torch.zeros((N, ref.shape[2], ref.shape[3], ref.shape[1]), device="cuda",
                      dtype=torch.bfloat16 if prec == "bf16" else torch.float32)
    auxd = nhwc_dev(aux, prec) if aux is not None else None
    ideq.debug_conv(kind, prec, use_tc, w32, N, Hin, Win, xin, out, auxd, epi)
    got = from_nhwc_dev(out)
    tol = 1e-5 if prec == "fp32" else 8e-3
    assert np.isfinite(got).all()
    assert rel_l2(got, ref) <= tol, (path, rel_l2(got, ref))
    assert_elementwise(got, ref, prec)


@pytest.mark.parametrize("kind,cin,cout,N,H,W,epi", [(0, 64, 128, 3, 8, 40, 2), (1, 128, 64, 3, 8, 40, 3),
                                                     (0, 128, 256, 1, 24, 24, 1), (1, 256, 128, 1, 24, 24, 3)])
def test_streamed_weight_layer_odd_tile_count(kind, cin, cout, N, H, W, epi):
    """Streamed-weight 3x3 layers (MODE 2: weights through a second TMA ring) with an odd number
    of 16x8 tiles and, for 24x24, a partial last tile row (zero-filled loads, clipped stores).
    Checked against the oracle layer, whole tensor and element by element."""
    torch = torch_cuda()
    from paper_2605_19705_b200 import ideq
    rng = np.random.default_rng(7 + kind)
    fn, wshape = KINDS[kind]
    w = rng.standard_normal(wshape(cin, cout)) * np.sqrt(1.0 / (cin * 4))
    x = rng.standard_normal((N, cin, H, W))
    w32 = w.astype(np.float32)
    xr, wr = bf16_round(x), bf16_round(w32)
    ref_acc = np.stack([fn(xr[n], wr) for n in range(N)])
    aux = auxr = None
    if epi in (2, 3):
        aux = rng.uniform(0.05, 2.0, ref_acc.shape) if epi == 3 else rng.standard_normal(ref_acc.shape)
        auxr = bf16_round(aux)
    ref = _epi_ref(ref_acc, epi, auxr)
    out = torch.zeros((N, ref.shape[2], ref.shape[3], ref.shape[1]), device="cuda", dtype=torch.bfloat16)
    ideq.debug_conv(kind, "bf16", True, w32, N, H, W, nhwc_dev(x, "bf16"), out,
                    nhwc_dev(aux, "bf16") if aux is not None else None, epi)
    got = from_nhwc_dev(out)
    assert np.isfinite(got).all()
    assert rel_l2(got, ref) <= 8e-3
    assert_elementwise(got, ref, "bf16")
