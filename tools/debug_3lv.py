import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_05982_b200 as vx
def run(n, frac_dense, dt, seed=5):
    g = torch.Generator(device="cuda"); g.manual_seed(seed)
    bits = 63 if dt == "u64" else 31
    idt = torch.int64 if dt == "u64" else torch.int32
    x = torch.randint(-2**bits, 2**bits - 1, (n,), dtype=idt, device="cuda", generator=g)
    k = int(n * frac_dense)
    x[:k] = x[:k] & ((1 << (bits - 20)) - 1)   # dense cluster near 0 -> deep recursion
    mn = torch.iinfo(idt).min
    ref = torch.sort(x ^ mn)[0] ^ mn
    xv = x.view(torch.uint64 if dt == "u64" else torch.uint32)
    st = vx.sort(xv, vx.SortConfig(seed=3))
    torch.cuda.synchronize()
    bad = (x != ref).nonzero()
    print(dt, n, frac_dense, "levels", st.max_depth, "pc", st.partition_calls, "base", st.base_case_calls,
          "fb", st.fallback_triggered, "bad", bad.numel(), flush=True)
    return bad.numel()
for dt in ("u64", "u32"):
    for n in (1 << 22, 1 << 24):
        for f in (0.5, 0.9):
            run(n, f, dt)
