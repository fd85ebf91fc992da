"""Workspace plan and sharding on one GPU (images are independent, PAPER
P:209 Alg. 1's "for each (y, x*)"):

- micro-batching: the network's activations are allocated for a micro-batch and a solve runs the
  network once per micro-batch; results equal the one-pass solve bit for bit, stop iteration
  included (per-image and GLOBAL_MAX rules, bf16 and fp32);
- sharding (the P-rank layout emulated by solving the shards one after another, SURVEY §4
  "Multi-GPU without a cluster"): per-image results do not depend on the shard, and under
  GLOBAL_MAX a shard never stops later than the whole batch (its max residual is <= the global
  max at every check), so shards run to the whole batch's stop iteration reproduce it exactly;
- the planner: an explicit byte budget fixes the micro-batch; a budget below one image fails
  with IDEQ_E_NOMEM.
"""
import numpy as np
import pytest

from paper_2605_19705_b200 import configs, synth
from paper_2605_19705_b200 import dist as dist_util
from tests.gpu_util import torch_cuda

pytestmark = pytest.mark.gpu


def _run(cfg, prob, precision, micro_batch=0, workspace_bytes=0, **pk):
    torch = torch_cuda()
    from paper_2605_19705_b200 import ideq
    s = ideq.Solver(cfg, prob["weights"], precision=precision, max_batch=len(prob["images"]),
                    micro_batch=micro_batch, workspace_bytes=workspace_bytes)
    s.set_operator(prob)
    plan = s.plan()
    xd = torch.tensor(np.ascontiguousarray(prob["x0"], dtype=np.float32)).cuda()
    yd = torch.tensor(np.ascontiguousarray(prob["y"], dtype=np.float32)).cuda()
    st, code, _ = s.solve(yd, xd, s.params(**pk))
    x = xd.cpu().numpy()
    s.close()
    return st, x, plan


def _same(a, b):
    for k in ("iters", "status", "residual"):
        assert np.array_equal(a[0][k], b[0][k]), k
    assert np.array_equal(a[1], b[1])


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
@pytest.mark.parametrize("name,pk", [("C3", dict(max_iter=6, tol=0.0)), ("C3", dict(max_iter=40, tol=1e-3)),
                                     ("C5", dict(max_iter=60, tol=5e-3, check_every=3)),
                                     ("C2", dict(max_iter=5, tol=0.0)), ("C4", dict(max_iter=5, tol=0.0))])
def test_micro_batched_equals_one_pass(name, pk, precision):
    kw = dict(C2=dict(H=32, W=48), C3=dict(H=32, W=48), C4=dict(H=32, W=32, tau=0.5 / 21),
              C5=dict(H=32, W=64))[name]
    cfg = configs.get(name, batch=5, **kw)
    prob = synth.make_problem(cfg)
    whole = _run(cfg, prob, precision, **pk)
    assert whole[2]["micro_batch"] == 5
    for mb in (2, 3):
        part = _run(cfg, prob, precision, micro_batch=mb, **pk)
        assert part[2]["micro_batch"] == {2: 2, 3: 3}[mb] or part[2]["micro_batch"] <= mb
        _same(whole, part)


def test_shards_reproduce_the_whole_batch_global_max():
    cfg = configs.get("C5", batch=6, H=32, W=64, max_iter=60, tol=5e-3, check_every=3)
    prob = synth.make_problem(cfg)
    whole_st, whole_x, _ = _run(cfg, prob, "bf16")
    k_star = int(whole_st["iters"].max())
    assert (whole_st["status"] == 0).all() and k_star < 60 and k_star % 3 == 0
    P = 3
    xs = []
    for r in range(P):
        idx = list(dist_util.shard(cfg["batch"], P, r))
        sub = synth.make_problem(configs.get("C5", batch=len(idx), H=32, W=64, max_iter=60, tol=5e-3,
                                             check_every=3), images=idx)
        st_own, _, _ = _run(cfg, sub, "bf16")
        assert int(st_own["iters"].max()) <= k_star        # a shard's max r <= the global max
        st_fix, x_fix, _ = _run(cfg, sub, "bf16", max_iter=k_star, tol=0.0)
        xs.append(x_fix)
    assert np.array_equal(np.concatenate(xs), whole_x)


def test_planner_budget():
    torch_cuda()
    from paper_2605_19705_b200 import ideq
    cfg = configs.get("C3", batch=8, H=32, W=32)
    prob = synth.make_problem(cfg)
    s = ideq.Solver(cfg, prob["weights"], precision="bf16", max_batch=8)
    full = s.plan()
    s.close()
    assert full["micro_batch"] == 8
    per_img = full["workspace_bytes"] // 8
    s = ideq.Solver(cfg, prob["weights"], precision="bf16", max_batch=8, workspace_bytes=3 * per_img + 1)
    p3 = s.plan()
    s.close()
    assert p3["micro_batch"] == 3 or p3["micro_batch"] == 2   # 8 images in 3 balanced passes of <= 3
    assert p3["workspace_bytes"] <= 3 * per_img
    with pytest.raises(ideq.IdeqError) as ei:
        ideq.Solver(cfg, prob["weights"], precision="bf16", max_batch=8, workspace_bytes=per_img // 2)
    assert ei.value.code == ideq.E_NOMEM
