L=paper_2205_05982_b200/lib
cp $L/libvxsort_b200.so /tmp/keep.so
for r in 1; do
  for v in ${VARIANTS:-A B C}; do
    cp $L/lib$v.so $L/libvxsort_b200.so
    for w in ${WL:-c2-u32-asc u64-uniform c3a c3f c2-f32-asc}; do
      echo -n "$v "; timeout 120 python tools/time_kernels.py --workload $w --reps 5 | cut -c1-${CUT:-330}
    done
  done
done
cp /tmp/keep.so $L/libvxsort_b200.so
