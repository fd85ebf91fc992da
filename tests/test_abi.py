"""CPU checks of the C-ABI boundary: the library builds, loads and exports every symbol
the headers in include/ declare; without a GPU it refuses to compute (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INCLUDE = os.path.join(ROOT, "include")


def _declared_symbols():
    names = set()
    for f in os.listdir(INCLUDE):
        if f.endswith(".h"):
            txt = open(os.path.join(INCLUDE, f)).read()
            names |= set(re.findall(r"IDEQ_API\s+[\w\s\*]+?\b(ideq_\w+)\s*\(", txt))
    return names


@pytest.fixture(scope="module")
def lib():
    from paper_2605_19705_b200 import build, ideq
    build.build()
    return ideq.load_library()


def test_headers_declare_the_boundary():
    names = _declared_symbols()
    for s in ["ideq_create", "ideq_set_operator", "ideq_solve", "ideq_destroy", "ideq_solve_host", "ideq_grad_g",
              "ideq_last_error", "ideq_get_nccl_id", "ideq_debug_conv"]:
        assert s in names


def test_library_exports_every_declared_symbol(lib):
    for s in _declared_symbols():
        assert hasattr(lib, s), s
    assert lib.ideq_abi_version() == 3


def test_python_binding_covers_the_abi():
    from paper_2605_19705_b200 import ideq
    assert set(ideq.SYMBOLS) == _declared_symbols()


def test_struct_layouts_match_header():
    """ctypes mirrors of the ABI structs have the C sizes (x86-64 SysV)."""
    from paper_2605_19705_b200 import ideq
    assert ctypes.sizeof(ideq.Params) == 11 * 4
    assert ctypes.sizeof(ideq.OperatorDesc) == 64  # 5 ints + 3 pointers (+pad) + int + pointer + float (+pad)
    assert ctypes.sizeof(ideq.ImageStat) == 20
    assert ctypes.sizeof(ideq.Dist) == 8 + 128
    assert ctypes.sizeof(ideq.NetDesc) == 56  # 9 ints + 4 pad + pointer + size_t
    assert ctypes.sizeof(ideq.Profile) == 4 * 6 * 8


def test_no_cpu_fallback_without_gpu(lib):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2605_19705_b200 import configs, ideq, synth
    cfg = configs.get("C1")
    prob = synth.make_problem(cfg)
    with pytest.raises(ideq.IdeqError) as ei:
        ideq.Solver(cfg, prob["weights"])
    assert ei.value.code == ideq.E_CUDA


def test_invalid_arguments_rejected_before_device_use(lib):
    from paper_2605_19705_b200 import configs, ideq, synth
    cfg = configs.get("C1")
    prob = synth.make_problem(cfg)
    with pytest.raises(ideq.IdeqError) as ei:
        ideq.Solver(cfg, prob["weights"][:-1])          # wrong blob size
    assert ei.value.code == ideq.E_INVALID
    bad = dict(cfg, net="unet4", widths=(32, 64, 128, 256), H=30)
    with pytest.raises(ideq.IdeqError) as ei:
        ideq.Solver(bad, np.zeros(10, np.float32))
    assert ei.value.code == ideq.E_INVALID
