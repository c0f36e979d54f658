"""vxs_sort inside a CUDA graph: a sort on a capturing
stream launches without any host round trip, so it can be captured once and
replayed; every replay must produce the oracle's output, and
vxs_workspace_status reads the device control block afterwards."""
import numpy as np
import pytest
import torch

import oracle
import paper_2205_05982_b200 as vx

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kt,n,desc", [("u64", 1_000_000, False), ("u32", 3_000_000, True), ("f32", 700_001, False),
                                       ("k128", 200_000, False), ("u64", 5_000, False), ("i16", 1, False)])
def test_sort_replays_from_a_cuda_graph(cuda, kt, n, desc):
    rng = np.random.default_rng(n)
    if kt == "k128":
        x = rng.integers(0, 2**64, (n, 2), dtype=np.uint64)
        x[:, 1] >>= np.uint64(50)
    elif kt == "f32":
        x = (rng.standard_normal(n) * 1e3).astype(np.float32)
        x[::97] = np.nan
    else:
        dt = {"u64": np.uint64, "u32": np.uint32, "i16": np.int16}[kt]
        info = np.iinfo(dt)
        x = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
    src = torch.from_numpy(x).cuda()
    buf = src.clone()
    ws = torch.empty(vx.workspace_bytes(n, kt), dtype=torch.uint8, device="cuda")
    cfg = vx.SortConfig(order=vx.Order(int(desc)), seed=5)
    ktarg = kt if kt == "k128" else None
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up outside capture (module load, pools)
        vx.sort(buf, cfg, key_type=ktarg, workspace=ws)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        vx.sort(buf, cfg, key_type=ktarg, workspace=ws)
    want, _ = oracle.sort(x, kt, descending=desc)
    for _ in range(3):
        buf.copy_(src)
        g.replay()
        torch.cuda.synchronize()
        assert buf.cpu().numpy().tobytes() == want.tobytes()
    st = vx.workspace_status(ws, n, kt)
    if n > vx.base_case_capacity(kt):
        assert st.max_depth >= 1 and st.keys_partitioned >= n


def test_graph_replay_is_faster_for_c1(cuda):
    """C1 (1e6 u64): the replayed graph beats the synchronising call (no host
    round trip, no per-kernel launch latency)."""
    from paper_2205_05982_b200 import workloads
    x, kt, _ = workloads.make("c1")
    src = torch.from_numpy(x).cuda()
    buf = src.clone()
    ws = torch.empty(vx.workspace_bytes(len(x), kt), dtype=torch.uint8, device="cuda")
    cfg = vx.SortConfig(seed=1)
    vx.sort(buf, cfg, workspace=ws)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        vx.sort(buf, cfg, workspace=ws)

    def timed(fn, reps=20):
        ts = []
        for _ in range(reps):
            buf.copy_(src)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts))
    t_call = timed(lambda: vx.sort(buf, cfg, workspace=ws))
    t_graph = timed(g.replay)
    print(f"C1: call {t_call:.4f} ms, graph replay {t_graph:.4f} ms")
    want, _ = oracle.sort(x, kt)
    assert buf.cpu().numpy().tobytes() == want.tobytes()
    assert t_graph < t_call
