#!/bin/bash
# Per-kernel timings over the BASELINE workloads (experiments; run on the GPU box).
for w in ${WL:-c2-u32-asc u64-uniform c2-f32-asc c2-u32-desc c3a c3c c3e c3f c4a c4b c1}; do
  timeout 120 python tools/time_kernels.py --workload $w --reps ${REPS:-5}
done
