import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_05982_b200 as vx
def run(lg, dt):
    n = 1 << lg
    g = torch.Generator(device="cuda"); g.manual_seed(5)
    if dt == "u32":
        x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
        ref = (torch.sort(x ^ torch.iinfo(torch.int32).min)[0] ^ torch.iinfo(torch.int32).min)
        x = x.view(torch.uint32)
        mn = torch.iinfo(torch.int32).min
        sx = lambda t: t.view(torch.int32)
    else:
        x = torch.randint(-2**63, 2**63 - 1, (n,), dtype=torch.int64, device="cuda", generator=g)
        ref = (torch.sort(x ^ torch.iinfo(torch.int64).min)[0] ^ torch.iinfo(torch.int64).min)
        x = x.view(torch.uint64)
        sx = lambda t: t.view(torch.int64)
    st = vx.sort(x, vx.SortConfig(seed=3))
    torch.cuda.synchronize()
    bad = (sx(x) != ref).nonzero()
    print(dt, lg, "levels", st.max_depth, "pc", st.partition_calls, "base", st.base_case_calls, "bad", bad.numel(), flush=True)
run(29, "u64"); run(29, "u64")
