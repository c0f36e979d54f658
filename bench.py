#!/usr/bin/env python3
"""bench.py -- the driver's measurement contract for the B200 sort.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload c2-u32-asc]

A STEP is one full sort (the hot path) of one synthetic batch already
resident in HBM.  Default workload (N=1) is BASELINE.json configs[1]'s first
case: 1e8 uint32 keys, uniform full range, ascending.  At N>1 (torchrun, one
rank per GPU, NCCL) the step is the distributed sample sort of 1e8 uint32
keys PER RANK (weak scaling).  Rank 0 prints one JSON line.

value   = whole-job Mkeys/s, device-timed with CUDA events (max over ranks)
e2e     = the same metric through the public host API (vxs_sort_host via
          paper_2205_05982_b200.sort(numpy)) from pinned host memory, H2D and
          D2H inside the timed region
roofline= dominant kernel's algorithmic bytes per launch / its event-timed
          average duration, against MEASURED_PEAKS.json's HBM copy bandwidth
cpu_baseline = the reference's own sort (oracle/_ref, compiled from
          /root/reference sources) on this host's cores, bounded sample.
Inputs (400 MB) exceed the 126 MB L2, and every step restores the unsorted
input with an untimed device copy first, which also evicts L2.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

KEYS_PER_CPU_INSTANCE = 10_000_000


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------- clocks ----
class ClockSampler:
    """Polls NVML every few ms on a background thread (SM clock, reasons)."""

    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
             0x100: "display_clocks_setting"}

    def __init__(self, index=0, period=0.005):
        self.samples = []
        self.reasons = 0
        self.period = period
        self.ok = False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            log("clock sampler unavailable:", e)
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                util = nv.nvmlDeviceGetUtilizationRates(self.h).gpu
                self.samples.append((mhz, r, util))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        busy = [s for s in self.samples if not (s[1] & 0x1)] or self.samples
        reasons = 0
        for s in busy:
            reasons |= s[1]
        names = [v for k, v in self.NAMES.items() if reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(s[0] for s in busy), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(busy)}


# ---------------------------------------------------------------- helpers ----
def torch_dtype(kt):
    import torch
    return {"u16": torch.uint16, "i16": torch.int16, "u32": torch.uint32, "i32": torch.int32,
            "f32": torch.float32, "u64": torch.uint64, "i64": torch.int64, "f64": torch.float64,
            "k128": torch.uint64, "kv64": torch.uint64}[kt]


def to_device(x, kt):
    import torch
    t = torch.from_numpy(x)
    return t.to("cuda")


def check_sorted_device(buf, kt, desc, src=None):
    """Device-side validation of a sorted result: non-decreasing in the
    order-transformed domain, and the same multiset fingerprint as the input."""
    import torch
    import paper_2205_05982_b200 as vx
    w = buf.clone()
    vx.transform(w, vx.Order(int(desc)), key_type=kt if kt in ("k128", "kv64") else None)
    kb = vx.KEY_BYTES[kt]
    if kb == 16:
        hi = w[:, 1].view(torch.int64) ^ torch.iinfo(torch.int64).min
        lo = w[:, 0].view(torch.int64) ^ torch.iinfo(torch.int64).min
        ok = bool(((hi[1:] > hi[:-1]) | ((hi[1:] == hi[:-1]) & (lo[1:] >= lo[:-1]))).all())
    else:
        sdt = {2: torch.int16, 4: torch.int32, 8: torch.int64}[kb]
        s = w.view(sdt) ^ torch.iinfo(sdt).min
        ok = bool((s[1:] >= s[:-1]).all())
    if src is not None:
        ok = ok and fingerprint(buf, kb) == fingerprint(src, kb)
    return ok


def fingerprint(t, kb):
    """Order-independent multiset fingerprint (sum and sum of squares of a
    64-bit mix of every key), computed on the device."""
    import torch
    if kb == 8 or kb == 16:
        w = t.reshape(-1).view(torch.int64)
    elif kb == 4:
        w = t.reshape(-1).view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    else:
        w = t.reshape(-1).view(torch.int16).to(torch.int64) & 0xFFFF
    if kb == 16:
        w = w.reshape(-1, 2)
        w = w[:, 0] * -7046029254386353131 + w[:, 1]
    h = w * -4658895280553007687
    h = h ^ (h >> 29)
    h = h * -7723592293110705685
    return int(h.sum()), int((h * h).sum())


def algorithmic_bytes(stats, n, kb):
    """Design bytes per sort: each level = hist (read) + scatter (read+write)
    over the keys it partitions; base case = read+write of every key."""
    kp = stats.keys_partitioned
    return {"k_hist": kp * kb, "k_scatter": 2 * kp * kb, "k_final": 2 * n * kb,
            "total": 3 * kp * kb + 2 * n * kb}


# ---------------------------------------------------------------- CPU leg ----
def cpu_reference_run(x, kt, desc, instances, n_each, reps):
    """Independent-instance throughput of the reference's own vexsort::sort
    (harness.cpp:316-358 threads mode) over `instances` host threads."""
    import ctypes
    import oracle
    use_ref = oracle.ref_available()
    okt = "k128" if kt == "kv64" else kt
    n_total = x.shape[0]
    bufs = []
    for i in range(instances):
        s = (i * n_each) % max(1, n_total - n_each + 1)
        bufs.append(np.ascontiguousarray(x[s:s + n_each]).copy())
    pristine = [b.copy() for b in bufs]
    if okt in ("f32", "f64"):
        for b in bufs + pristine:  # the reference rejects NaN (driver.hpp:176-180)
            b[np.isnan(b)] = np.inf
    times = []
    for r in range(reps):
        for b, p in zip(bufs, pristine):
            b[...] = p
        ptrs = (ctypes.c_void_p * instances)(*[b.ctypes.data for b in bufs])
        t0 = time.perf_counter()
        if use_ref:
            rc = oracle.ref().ref_sort_instances(ptrs, instances, n_each, oracle.KEY_CODE[okt], int(desc), 1)
            assert rc == 0, oracle.ref().ref_last_error()
        else:
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(instances) as ex:
                list(ex.map(lambda b: oracle.lib().vxo_sort(b.ctypes.data, n_each, oracle.KEY_CODE[okt],
                                                             int(desc), 1, None), bufs))
        times.append(time.perf_counter() - t0)
    return times, ("reference" if use_ref else "port")


def cpu_baseline(x, kt, desc):
    cores = os.cpu_count() or 1
    n_each = min(KEYS_PER_CPU_INSTANCE, x.shape[0])
    times, kind = cpu_reference_run(x, kt, desc, cores, n_each, reps=2)
    t = statistics.median(times)
    one, _ = cpu_reference_run(x, kt, desc, 1, n_each, reps=1)
    return {"value": round(cores * n_each / t / 1e6, 2), "unit": "Mkeys/s", "cores": cores, "kind": kind,
            "sample": f"{cores} independent instances x {n_each} keys of the same workload "
                      f"(vexsort::sort, harness threads mode); median of 2 reps",
            "single_core_mkeys_s": round(n_each / one[0] / 1e6, 2)}


# ---------------------------------------------------------------- GPU leg ----
def gpu_time_sorts(buf, src, ws, kt, desc, steps, warmup, seed=1, profile=False, dist_sync=None):
    import torch
    import paper_2205_05982_b200 as vx
    cfg = vx.SortConfig(order=vx.Order(int(desc)), seed=seed)
    ktarg = kt if kt in ("k128", "kv64") else None
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        buf.copy_(src)
        vx.sort(buf, cfg, key_type=ktarg, workspace=ws)
    torch.cuda.synchronize()
    if profile:
        vx.profile_reset()
        vx.profile_enable(True)
    times = []
    launches = 0
    last = None
    for _ in range(steps):
        buf.copy_(src)  # restore unsorted input (untimed; also evicts L2)
        if dist_sync:
            dist_sync()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        st = vx.sort(buf, cfg, key_type=ktarg, workspace=ws)
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
        launches += st.kernel_launches
        last = st
    prof = None
    if profile:
        prof = vx.profile_read()
        vx.profile_enable(False)
    return times, launches, last, prof


def e2e_host(x, kt, desc, steps):
    """Public host API end to end: pinned host keys -> vxs_sort_host (H2D,
    sort, D2H inside) -> sorted host keys."""
    import torch
    import paper_2205_05982_b200 as vx
    pinned = torch.empty(x.shape, dtype=torch_dtype(kt)).pin_memory()
    host = pinned.numpy()
    cfg = vx.SortConfig(order=vx.Order(int(desc)), seed=1)
    ktarg = kt if kt in ("k128", "kv64") else None
    host[...] = x
    vx.sort(host, cfg, key_type=ktarg)  # warm-up (pool, module load)
    times = []
    for _ in range(steps):
        host[...] = x
        t0 = time.perf_counter()
        vx.sort(host, cfg, key_type=ktarg)
        times.append(time.perf_counter() - t0)
    return times, x.nbytes


def roofline(prof, stats, n, kb, peak):
    bytes_ = algorithmic_bytes(stats, n, kb)
    agg = {}
    for name, (l, ms) in prof.items():  # per-level entries "k_scatter@L0" -> "k_scatter"
        base = name.split("@")[0]
        a = agg.setdefault(base, [0, 0.0])
        a[0] += l
        a[1] += ms
    prof = {k: tuple(v) for k, v in agg.items()}
    fin_l = sum(v[0] for k, v in prof.items() if k.startswith("k_final") and k != "k_final_phase")
    fin_ms = sum(v[1] for k, v in prof.items() if k.startswith("k_final") and k != "k_final_phase")
    if "k_final_phase" in prof:  # wall time of the (partly concurrent) class launches
        fin_ms = prof["k_final_phase"][1]
    per_kernel = {}
    for k in ("k_hist", "k_scatter"):
        if k in prof:
            l, ms = prof[k]
            per_kernel[k] = {"launches": l, "ms": ms, "bytes_per_sort": bytes_[k]}
    if fin_l:
        # the base case is one phase launched per size class (most classes
        # are near-empty): count it as one launch per sort so the bytes of the
        # whole phase are divided by the whole phase's time
        sorts = prof.get("k_final_phase", prof.get("k_init", (fin_l, 0.0)))[0]
        per_kernel["k_final"] = {"launches": sorts, "ms": fin_ms, "bytes_per_sort": bytes_["k_final"],
                                 "class_launches": fin_l}
    return per_kernel


def ncu_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:  # noqa: BLE001
            return None
    return None


def run_single(args):
    import torch
    import paper_2205_05982_b200 as vx
    from paper_2205_05982_b200 import workloads
    peak, peak_src = measured_peaks()
    x, kt, desc = workloads.make(args.workload, n=args.n)
    n = x.shape[0]
    kb = vx.KEY_BYTES[kt]
    src = to_device(x, kt)
    buf = torch.empty_like(src)
    ws = torch.empty(vx.workspace_bytes(n, kt), dtype=torch.uint8, device="cuda")
    # correctness gate before timing
    buf.copy_(src)
    vx.sort(buf, vx.SortConfig(order=vx.Order(int(desc)), seed=1),
            key_type=kt if kt in ("k128", "kv64") else None, workspace=ws)
    torch.cuda.synchronize()
    assert check_sorted_device(buf, kt, desc, src), "sorted-output validation failed"
    with ClockSampler() as clk:
        times, launches, st, _ = gpu_time_sorts(buf, src, ws, kt, desc, args.steps, args.warmup)
    ms = statistics.mean(times)
    # per-kernel breakdown from separate profiled steps (the per-launch CUDA
    # events are kept out of the timed region)
    _, _, _, prof = gpu_time_sorts(buf, src, ws, kt, desc, args.steps, 1, profile=True)
    steps = args.steps
    # per-kernel breakdown (events around every launch in the timed steps)
    per = roofline(prof, st, n, kb, peak)
    dom_name = max(per, key=lambda k: per[k]["ms"])
    dom = per[dom_name]
    launches_per_sort = dom["launches"] / steps
    bytes_per_launch = dom["bytes_per_sort"] / launches_per_sort
    avg_launch_ms = dom["ms"] / dom["launches"]
    achieved = bytes_per_launch / (avg_launch_ms * 1e-3) / 1e9
    ncu = ncu_traffic()
    traffic = None
    if ncu and ncu.get("workload") == args.workload and dom_name in ncu.get("kernels", {}):
        traffic = ncu["kernels"][dom_name].get("dram_bytes_per_launch")
    total_alg = algorithmic_bytes(st, n, kb)["total"]
    if args.no_e2e:  # profiling runs only: keep the launch list to the device-resident sort
        e2e_t, hbytes = [float("nan")], 0
    else:
        e2e_t, hbytes = e2e_host(x, kt, desc, min(steps, 5))
    e2e_s = statistics.median(e2e_t)
    line = {
        "metric": "Mkeys/s sorted (in-memory key sort)",
        "value": round(n / (ms * 1e-3) / 1e6, 2),
        "unit": "Mkeys/s",
        "n_gpus": 1,
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": kt,
        "data": "synthetic (seeded SplitMix64; BASELINE.json config shapes)",
        "config": {"workload": args.workload, "n": n, "key_type": kt, "order": "desc" if desc else "asc",
                   "key_bytes": kb, "parallelism": "single GPU",
                   "l2": f"inputs ({n * kb / 1e6:.0f} MB) larger than L2 (126 MB); untimed restore copy per step"},
        "gb_per_s_sorted": round(n * kb / (ms * 1e-3) / 1e9, 2),
        "levels": st.max_depth,
        "design_hbm_frac": round(total_alg / (ms * 1e-3) / 1e9 / peak, 4),
        "ideal_one_pass_frac": round(2 * n * kb / (ms * 1e-3) / 1e9 / peak, 4),
        "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "algorithmic_bytes_per_launch": int(bytes_per_launch),
                     "avg_launch_ms": round(avg_launch_ms, 4), "peak_source": peak_src},
        "kernels": {k: {"launches": v[0], "ms_per_step": round(v[1] / steps, 4)} for k, v in prof.items()},
        "e2e": {"value": round(n / e2e_s / 1e6, 2), "unit": "Mkeys/s", "h2d_bytes_per_step": hbytes,
                "d2h_bytes_per_step": hbytes, "ms_per_step": round(e2e_s * 1e3, 3),
                "api": "paper_2205_05982_b200.sort(numpy pinned) -> vxs_sort_host"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "sort_stats": {"max_depth": st.max_depth, "partition_calls": st.partition_calls,
                       "base_case_calls": st.base_case_calls, "keys_partitioned": st.keys_partitioned,
                       "fallback_triggered": st.fallback_triggered},
    }
    if not args.no_extras:
        extra = {}
        for wl in args.extras.split(","):
            if not wl or wl == args.workload:
                continue
            xe, kte, de = workloads.make(wl)
            ne = xe.shape[0]
            se = to_device(xe, kte)
            be = torch.empty_like(se)
            wse = torch.empty(vx.workspace_bytes(ne, kte), dtype=torch.uint8, device="cuda")
            be.copy_(se)
            vx.sort(be, vx.SortConfig(order=vx.Order(int(de)), seed=1),
                    key_type=kte if kte in ("k128", "kv64") else None, workspace=wse)
            torch.cuda.synchronize()
            okx = check_sorted_device(be, kte, de, se)
            te, _, ste, _ = gpu_time_sorts(be, se, wse, kte, de, 3, 2)
            _, _, _, pre = gpu_time_sorts(be, se, wse, kte, de, 3, 1, profile=True)
            mse = statistics.mean(te)
            kbe = vx.KEY_BYTES[kte]
            pe = roofline(pre, ste, ne, kbe, peak)
            sc = pe.get("k_scatter")
            extra[wl] = {"mkeys_s": round(ne / (mse * 1e-3) / 1e6, 2), "ms": round(mse, 3), "n": ne,
                         "gb_per_s_sorted": round(ne * kbe / (mse * 1e-3) / 1e9, 2), "validated": okx,
                         "levels": ste.max_depth,
                         "design_hbm_frac": round(algorithmic_bytes(ste, ne, kbe)["total"] / (mse * 1e-3) / 1e9
                                                  / peak, 4),
                         "scatter_frac": (round(sc["bytes_per_sort"] / (sc["ms"] / 3 * 1e-3) / 1e9 / peak, 4)
                                          if sc else None),
                         "kernels_ms": {k: round(v[1] / 3, 4) for k, v in pre.items()}}
            del se, be, wse
            torch.cuda.empty_cache()
        line["extra"] = extra
    if not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(x, kt, desc)
    return line


def run_reference(args):
    from paper_2205_05982_b200 import workloads
    x, kt, desc = workloads.make(args.workload, n=args.n)
    cores = os.cpu_count() or 1
    n_each = min(KEYS_PER_CPU_INSTANCE, x.shape[0])
    cpu_reference_run(x, kt, desc, cores, n_each, reps=max(1, args.warmup))
    times, kind = cpu_reference_run(x, kt, desc, cores, n_each, reps=args.steps)
    t = statistics.mean(times)
    val = round(cores * n_each / t / 1e6, 2)
    return {
        "impl": "reference",
        "metric": "Mkeys/s sorted (in-memory key sort)",
        "value": val, "unit": "Mkeys/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": kt, "data": "synthetic (seeded SplitMix64; BASELINE.json config shapes)",
        "config": {"workload": args.workload, "n": int(x.shape[0]), "key_type": kt,
                   "order": "desc" if desc else "asc", "parallelism": f"{cores} host threads"},
        "cpu_baseline": {"value": val, "unit": "Mkeys/s", "cores": cores, "kind": kind,
                         "sample": f"each step: {cores} independent vexsort::sort instances x {n_each} keys "
                                   f"of the workload (harness threads mode, harness.cpp:316-358)"},
        "e2e": {"value": val, "unit": "Mkeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def run_distributed(args):
    import torch
    import torch.distributed as dist
    import paper_2205_05982_b200 as vx
    from paper_2205_05982_b200 import workloads
    from paper_2205_05982_b200.dist import dist_sort
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peak, _ = measured_peaks()
    x, kt, desc = workloads.make(args.workload, n=args.n, seed=1 + rank)
    n = x.shape[0]
    kb = vx.KEY_BYTES[kt]
    src = to_device(x, kt)
    order = vx.Order(int(desc))
    for _ in range(args.warmup):
        out = dist_sort(src, order=order, key_type=kt, exchange=args.exchange, copy_out=False)
    torch.cuda.synchronize()
    # validation: local sortedness + boundary monotonicity + global count
    ok = check_sorted_device(out, kt, desc)
    cnt = torch.tensor([out.shape[0]], device="cuda", dtype=torch.int64)
    dist.all_reduce(cnt)
    ok = ok and int(cnt) == n * world
    times = []
    stream = torch.cuda.current_stream()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            dist.barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            out = dist_sort(src, order=order, key_type=kt, exchange=args.exchange, copy_out=False)
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
    t = torch.tensor([statistics.mean(times)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    okt = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    ms = float(t)
    # one untimed profiled step: our kernel launches per step + dominant-kernel roofline
    dist.barrier()
    vx.profile_reset()
    vx.profile_enable(True)
    out = dist_sort(src, order=order, key_type=kt, exchange=args.exchange, copy_out=False)
    torch.cuda.synchronize()
    prof = vx.profile_read()
    vx.profile_enable(False)
    launches = sum(v[0] for v in prof.values())
    sc = [(l, m) for k, (l, m) in prof.items() if k.split("@")[0] == "k_scatter"]
    sc_l, sc_ms = sum(l for l, _ in sc), sum(m for _, m in sc)
    achieved = (2 * n * kb) / ((sc_ms / max(sc_l, 1)) * 1e-3) / 1e9 if sc_l else 0.0
    ach = torch.tensor([achieved], device="cuda", dtype=torch.float64)
    dist.all_reduce(ach, op=dist.ReduceOp.MIN)
    # e2e through the public API at N GPUs: pinned host keys -> H2D -> dist_sort -> D2H, max over ranks
    host = torch.empty(src.shape, dtype=src.dtype).pin_memory()
    host.copy_(src.cpu())
    dev_in = torch.empty_like(src)
    host_out = torch.empty((2 * n,) + tuple(src.shape[1:]), dtype=src.dtype).pin_memory()
    e2e_times, d2h_bytes = [], 0
    for _ in range(min(args.steps, 5)):
        dist.barrier()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        dev_in.copy_(host, non_blocking=True)
        res = dist_sort(dev_in, order=order, key_type=kt, exchange=args.exchange, copy_out=False)
        m = min(res.shape[0], host_out.shape[0])
        host_out[:m].copy_(res[:m], non_blocking=True)
        b.record(stream)
        torch.cuda.synchronize()
        e2e_times.append(a.elapsed_time(b))
        d2h_bytes = m * kb
    te = torch.tensor([statistics.median(e2e_times)], device="cuda", dtype=torch.float64)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te)
    line = None
    if rank == 0:
        line = {
            "metric": "Mkeys/s sorted (in-memory key sort)",
            "value": round(world * n / (ms * 1e-3) / 1e6, 2), "unit": "Mkeys/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": kt,
            "data": "synthetic (seeded SplitMix64 per rank; BASELINE.json config shapes)",
            "config": {"workload": args.workload + " (per rank)", "n_per_rank": n, "key_type": kt,
                       "parallelism": f"distributed sample sort x{world} (NCCL all-gather of samples/counts; "
                                              f"{args.exchange} key exchange)"},
            "validated": bool(int(okt)),
            "gb_per_s_sorted": round(world * n * kb / (ms * 1e-3) / 1e9, 2),
            "clocks": clk.summary(),
            "peak_hbm_gbs": peak,
            "roofline": {"bound": "hbm", "kernel": "k_scatter", "achieved": round(float(ach), 1), "peak": peak,
                         "unit": "GB/s", "frac": round(float(ach) / peak, 4) if peak else None, "traffic": None,
                         "note": "min over ranks; 2*n_local*key_bytes per launch / mean launch time"},
            "e2e": {"value": round(world * n / (e2e_ms * 1e-3) / 1e6, 2), "unit": "Mkeys/s",
                    "h2d_bytes_per_step": n * kb, "d2h_bytes_per_step": d2h_bytes, "ms_per_step": round(e2e_ms, 3),
                    "api": "pinned host keys per rank -> H2D -> dist_sort -> D2H (max over ranks)"},
            "gpu_launches": int(launches) * args.steps,
        }
    dist.destroy_process_group()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2-u32-asc")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--extras", default="u64-uniform,c2-f32-asc")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-API e2e leg (ncu launch lists only)")
    ap.add_argument("--force-dist", action="store_true", help="run the distributed path even at world size 1 (tests)")
    ap.add_argument("--exchange", default="fused", choices=["fused", "nccl"],
                    help="distributed key exchange: fused partition+P2P stores (default) or NCCL all-to-all")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(run_reference(args)), flush=True)
        return
    if world > 1 or args.force_dist:
        line = run_distributed(args)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    print(json.dumps(run_single(args)), flush=True)


if __name__ == "__main__":
    main()
