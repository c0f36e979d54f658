#!/bin/bash
# A/B(/C) timing of library builds on one box (experiments): alternates
# lib/lib{A,B,C}.so into place and times WL workloads with each.
L=paper_2205_05982_b200/lib
for r in 1 2; do
  for v in ${VARIANTS:-A B}; do
    cp $L/lib$v.so $L/libvxsort_b200.so
    for w in ${WL:-u64-uniform}; do
      echo -n "$v "; timeout 120 python tools/time_kernels.py --workload $w --reps ${REPS:-5} | cut -c1-${CUT:-150}
    done
  done
done
cp $L/libA.so $L/libvxsort_b200.so
