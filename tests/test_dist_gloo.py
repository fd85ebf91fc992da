"""World-size-2 gloo tests (CPU) of the data-parallel logic:
sharding, ncclUniqueId-style object broadcast, and the GLOBAL_MAX stop rule: the sharded
run with an all-reduced max residual stops on the same iteration and produces the same
iterates as the unsharded oracle (BASELINE C5 rule, reading Q17)."""
import os
import socket

import numpy as np
import pytest

from paper_2605_19705_b200 import dist as pdist


def test_shard_partitions_every_batch():
    for n in (1, 7, 32, 512):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                sh = pdist.shard(n, world, r)
                seen += list(sh)
                assert len(sh) in (n // world, n // world + 1)
            assert seen == list(range(n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import solver
        from paper_2605_19705_b200 import configs, synth
        # object broadcast (the path the ncclUniqueId takes)
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == bytes(range(128))

        cfg = configs.get("C5", batch=4, H=32, W=32, widths=(8, 8, 8, 8), ksize=9, ksigma=1.6,
                          check_every=3, tol=2e-3, max_iter=40)
        mine = list(pdist.shard(cfg["batch"], world, rank))
        prob = synth.make_problem(cfg, images=mine)
        net = solver.make_net(cfg, prob["weights"])
        fids = solver.make_fidelities(cfg, prob)

        def allreduce_max(v):
            t = torch.tensor([v], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())

        # per-rank loop: identical arithmetic to the oracle, stop decision via the collective
        xc = [x.astype(np.float64) for x in prob["x0"]]
        xp = [x.copy() for x in xc]
        iters = [0] * len(mine)
        stop_at = None
        for k in range(cfg["max_iter"]):
            rs = []
            for b in range(len(mine)):
                xn = solver.ideq_step(xc[b], xp[b], net, fids[b], cfg["lam"], cfg["tau"], cfg["beta"], cfg["step"])
                rs.append(solver.residual(xn, xc[b]))
                xp[b], xc[b] = xc[b], xn
                iters[b] = k + 1
            if (k + 1) % cfg["check_every"] == 0:
                if pdist.global_stop(max(rs) if rs else -1.0, cfg["tol"], allreduce_max):
                    stop_at = k + 1
                    break
        q.put((rank, mine, [x.tolist() for x in xc], iters, stop_at))
    finally:
        dist.destroy_process_group()


def test_global_max_rule_sharded_equals_unsharded():
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    from oracle import solver
    from paper_2605_19705_b200 import configs, synth
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = configs.get("C5", batch=4, H=32, W=32, widths=(8, 8, 8, 8), ksize=9, ksigma=1.6,
                      check_every=3, tol=2e-3, max_iter=40)
    prob = synth.make_problem(cfg)
    ref = solver.solve_config(cfg, prob)
    stops = {r[4] for r in res}
    assert len(stops) == 1                                  # every rank took the same decision
    for rank, mine, xs, iters, stop_at in res:
        for j, i in enumerate(mine):
            assert iters[j] == ref["iters"][i]
            assert np.array_equal(np.array(xs[j]), ref["x"][i])
    assert stop_at == ref["iters"][0] and stop_at % cfg["check_every"] == 0
