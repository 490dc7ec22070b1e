"""Multi-GPU full-gradient design, checked on CPU with torch.distributed gloo
(world size 2 and 4): each rank takes its split range from the library's
shard plan (halp_shard_plan, the same host code the NCCL path uses),
computes its subtree root in the device's MIRROR order, all-gathers the
roots, and finishes the tree.  The gradient and loss must be bit-identical
to the single-process pass, for every world size -- the property that makes
the NCCL-sharded K1 GPU-count invariant."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import torch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    import paper_1803_03383_b200 as H

    n, d, C, dtype = case
    rng = np.random.default_rng(5)
    X = rng.standard_normal((n, d)).astype(np.float32)
    w = rng.standard_normal(d * C) * 0.1
    if C == 1:
        obj = O.OracleObjective(X, y=rng.standard_normal(n), l2=1e-3)
    else:
        obj = O.OracleObjective(X, labels=rng.integers(0, C, n), num_classes=C, l2=1e-3)
    plan = H.oracle_plan_for(n, d, C, dtype)
    sp = H.shard_plan(n, d, C, {"f64": 0, "f32": 1, "bf16": 2}[dtype], world, rank)
    assert sp["splits"] == plan["fg_splits"]
    mine = torch.from_numpy(obj.split_subtree(w, plan, sp["split_begin"], sp["split_end"]))
    bufs = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(bufs, mine)
    g, loss = obj.finalize(w, torch.stack(bufs).numpy())
    if rank == 0:
        g1 = obj.full_gradient(w, plan=plan)
        l1 = obj.loss_value(w, plan=plan)
        q.put((bool(np.array_equal(g, g1)), loss == l1))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", [(3000, 40, 1, "f32"), (2500, 33, 3, "f32")])
def test_sharded_fullgrad_bit_identical(world, case):
    from paper_1803_03383_b200 import build

    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert res == (True, True)
