"""The fused distributed exchange end to end in two processes sharing cuda:0:
dist_sort(exchange="fused") with the gloo backend over CUDA tensors (NCCL
refuses two ranks on one GPU).  Each rank's partition kernel stores its
segments into the other process's receive window through a CUDA IPC mapping;
no kernel waits on another process (ordering is the host collectives').
The concatenated rank outputs must equal the oracle's sort."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2205_05982_b200 import Order
    from paper_2205_05982_b200.dist import dist_sort
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        res = []
        for ci, (kt, desc, n) in enumerate([("u64", False, 400_000), ("i32", True, 300_000), ("u64", False, 900_000)]):
            rng = np.random.default_rng(40 + 7 * rank + ci)
            dt = {"u64": np.uint64, "i32": np.int32}[kt]
            info = np.iinfo(dt)
            x = rng.integers(info.min, info.max, n + 1000 * rank, dtype=dt, endpoint=True)
            out = dist_sort(torch.from_numpy(x).cuda(), order=Order(int(desc)), key_type=kt, exchange="fused")
            torch.cuda.synchronize()
            res.append((ci, x, out.cpu().numpy()))
        dist.barrier()
        q.put((rank, res))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))


def test_dist_sort_fused_two_processes(cuda):
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(got[r], str), got[r]
    cases = [("u64", False), ("i32", True), ("u64", False)]
    for ci, (kt, desc) in enumerate(cases):
        allin = np.concatenate([got[r][ci][1] for r in range(world)])
        out = np.concatenate([got[r][ci][2] for r in range(world)])
        want, _ = oracle.sort(allin, kt, descending=desc)
        assert out.tobytes() == want.tobytes(), (kt, desc)
