import sys, json
sys.path.insert(0, '.')
import bench
peak, _ = bench.measured_peaks()
for kt in ("u32", "u64"):
    r = bench.time_partition(kt, peak)
    r.pop("reference_cpu_1core", None)
    print(kt, r)
