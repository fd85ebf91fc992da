"""fp64 CPU oracle for the i-DEQ inference hot path (arXiv 2605.19705).

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import or run
anything in this package. The product path (``paper_2605_19705_b200``'s CUDA
library and its binding) never imports it, and this package never imports the
product path: the two share no code. Inputs come from
``paper_2605_19705_b200.synth`` (seeded generators, no method arithmetic).

Plain and slow on purpose: every function follows the paper's definition or
algorithm step by step in float64, with numpy matmul / FFT as library
primitives, and cites the passage it follows ("P:n" = /root/reference/PAPER.md
line n, "S:n" = SPEC.md line n, "Qn" = a reading listed in DESIGN.md).

Pins (tests/test_oracle_pins.py) tie every function to something other than
itself. Parity status per function is in DESIGN.md; the full nonlinear U-Net
trajectories are pinned only by composition ("parity unpinned" beyond that).
"""
from . import nets, operators, solver  # noqa: F401
