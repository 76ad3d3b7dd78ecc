"""World-size-2 gloo tests (CPU) of the data-parallel host logic: the NCCL unique id travels
from rank 0 to every rank, timing is the max over ranks, and averaging equal shards equals
the concatenated batch (DESIGN Q9)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1912_06680_b200 import dist as pdist
    payload = bytes(range(128)) if rank == 0 else None
    got = pdist.share_bytes(payload, 128, "cpu")
    mx = pdist.max_over_ranks(float(rank + 1) * 3.5, "cpu")
    # DP average of per-rank gradients with gloo (host-side reference of ncclAvg)
    g = torch.full((5,), float(rank + 1))
    dist.all_reduce(g)
    g /= world
    q.put((rank, got, mx, g.tolist()))
    dist.destroy_process_group()


def test_gloo_world2_host_logic():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got, mx, g in res:
        assert got == bytes(range(128))
        assert mx == 7.0
        assert np.allclose(g, 1.5)


def test_single_process_is_passthrough():
    from paper_1912_06680_b200 import dist as pdist
    assert pdist.share_bytes(b"abc", 3, "cpu") == b"abc"
    assert pdist.max_over_ranks(2.5, "cpu") == 2.5
    assert pdist.make_comm("cpu") is None
