import torch, time
n = 100_000_000
d = torch.empty(n, dtype=torch.int32, device="cuda").random_()
h = torch.empty(n, dtype=torch.int32).pin_memory()
a = torch.empty(1 << 28, dtype=torch.int32, device="cuda"); b = torch.empty_like(a)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(busy_iters, nsplit=1):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s2):
        for _ in range(busy_iters): b.copy_(a)
    with torch.cuda.stream(s1):
        e0.record()
        step = n // nsplit
        for i in range(nsplit):
            h[i*step:(i+1)*step].copy_(d[i*step:(i+1)*step], non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)
for _ in range(2): run(0)
print("D2H alone       ", [round(run(0), 2) for _ in range(3)])
print("D2H alone 64 pcs", [round(run(0, 64), 2) for _ in range(3)])
print("D2H + 3 copies (1 GiB each way, ~1 ms)", [round(run(3), 2) for _ in range(3)])
print("D2H + 20 copies (~7 ms)", [round(run(20), 2) for _ in range(3)])
