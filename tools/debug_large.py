import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_05982_b200 as vx
for lg in [int(a) for a in sys.argv[1:]]:
    n = 1 << lg
    g = torch.Generator(device="cuda"); g.manual_seed(5)
    x = torch.randint(-2**63, 2**63 - 1, (n,), dtype=torch.int64, device="cuda", generator=g).view(torch.uint64)
    ref = torch.sort(x.view(torch.int64) ^ torch.iinfo(torch.int64).min)[0] ^ torch.iinfo(torch.int64).min
    st = vx.sort(x, vx.SortConfig(seed=3))
    torch.cuda.synchronize()
    bad = (x.view(torch.int64) != ref).nonzero()
    print(lg, "levels", st.max_depth, "partition_calls", st.partition_calls, "base", st.base_case_calls,
          "mismatches", bad.numel(), "first", bad[:3].flatten().tolist() if bad.numel() else None, flush=True)
    if bad.numel():
        i = int(bad[0])
        print("  got", x[i-3:i+5].tolist())
        print("  ref", ref.view(torch.uint64)[i-3:i+5].tolist())
    del x, ref
    torch.cuda.empty_cache()
