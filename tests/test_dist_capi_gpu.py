"""The distributed sample sort behind the C ABI (vxs_dist_sort),
checked against the oracle:

* world 1 through a native NCCL communicator (vxs_nccl_comm_create) and
  through no communicator at all, both exchanges;
* two processes sharing cuda:0 with the library's host all-gather callback
  (NCCL refuses two ranks on one GPU): every rank's partition kernel stores
  its segments into the other process's IPC-mapped window; the rank outputs,
  concatenated, must equal the oracle's sort of the union.  Covers uneven and
  empty ranks, window growth across calls, 16/32/64/128-bit and float keys."""
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


def _keys(kt, n, seed):
    rng = np.random.default_rng(seed)
    if kt == "k128":
        x = np.empty((n, 2), dtype=np.uint64)
        x[:, 0] = rng.integers(0, 2**64, n, dtype=np.uint64)
        x[:, 1] = rng.integers(0, 1 << 12, n, dtype=np.uint64)  # many hi ties
        return x
    if kt in ("f32", "f64"):
        x = (rng.standard_normal(n) * 1e3).astype(np.float32 if kt == "f32" else np.float64)
        x[::101] = np.nan
        x[1::97] = -0.0
        x[2::89] = 0.0
        return x
    dt = {"u16": np.uint16, "i32": np.int32, "u64": np.uint64}[kt]
    info = np.iinfo(dt)
    return rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)


CASES = [("u64", False, 300_000), ("i32", True, 250_000), ("f32", False, 200_000), ("u16", False, 90_000),
         ("k128", True, 120_000), ("u64", False, 1_200_000)]  # (the last one grows the window)


def test_dist_capi_world1(cuda):
    import torch.distributed as dist
    from paper_2205_05982_b200 import Order
    from paper_2205_05982_b200.dist import NativeDist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        for comm in ("nccl", "host"):
            nd = NativeDist(comm=comm)
            for ci, (kt, desc, n) in enumerate(CASES):
                x = _keys(kt, n, 11 + ci)
                for exch in ("fused", "nccl"):
                    out, st = nd.sort(torch.from_numpy(x).cuda(), order=Order(int(desc)),
                                      key_type=kt if kt == "k128" else None, exchange=exch)
                    torch.cuda.synchronize()
                    want, _ = oracle.sort(x, kt, descending=desc)
                    assert out.cpu().numpy().tobytes() == want.tobytes(), (comm, kt, desc, exch)
                    assert st.kernel_launches > 0
            recv, sent = nd.last_counts()
            assert recv == [CASES[-1][2]] and sent == [CASES[-1][2]]
            nd.close()
    finally:
        dist.destroy_process_group()


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2205_05982_b200 import Order
    from paper_2205_05982_b200.dist import NativeDist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        nd = NativeDist(comm="host")
        res = []
        for ci, (kt, desc, n) in enumerate(CASES + [("u64", False, 0)]):
            # uneven ranks; the last case leaves rank 1 empty
            nr = n + 3000 * rank if ci < len(CASES) else (50_000 if rank == 0 else 0)
            x = _keys(kt, nr, 40 + 7 * rank + ci)
            out, _ = nd.sort(torch.from_numpy(x).cuda(), order=Order(int(desc)),
                             key_type=kt if kt == "k128" else None)
            torch.cuda.synchronize()
            res.append((ci, x, out.cpu().numpy().copy(), nd.last_counts()))
        nd.close()
        dist.barrier()
        q.put((rank, res))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))


def test_dist_capi_two_processes(cuda):
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(got[r], str), got[r]
    for ci, (kt, desc, _) in enumerate(CASES + [("u64", False, 0)]):
        allin = np.concatenate([got[r][ci][1] for r in range(world)])
        out = np.concatenate([got[r][ci][2] for r in range(world)])
        want, _ = oracle.sort(allin, kt, descending=desc)
        assert out.tobytes() == want.tobytes(), (kt, desc)
        recv, _ = got[0][ci][3]
        assert recv == [len(got[r][ci][2]) for r in range(world)]
        assert sum(recv) == len(allin)


def test_dist_capi_cpp_host(cuda, tmp_path):
    """A C++ host (tests/cpp/dist_sort_test.cpp) drives vexsort::DistSorter:
    world 1 with a native NCCL communicator and without, then two forked
    processes on one GPU with a shared-memory host all-gather; every result is
    checked against std::sort."""
    import shutil
    import subprocess
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib_dir = os.path.join(root, "paper_2205_05982_b200", "lib")
    exe = tmp_path / "dist_sort_test"
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(root, "include"), "-I", "/usr/local/cuda/include",
                        os.path.join(root, "tests", "cpp", "dist_sort_test.cpp"), "-o", str(exe), "-L", lib_dir,
                        "-lvxsort_b200", "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib_dir}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    for mode in ("world1", "fork2"):
        r = subprocess.run([str(exe), mode], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and r.stdout.strip().endswith("ok"), (mode, r.returncode, r.stdout, r.stderr)
