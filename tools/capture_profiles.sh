#!/bin/bash
# Round-tagged evidence for profiles/: bench line, ncu launch list, ncu --set full
# summaries (u64, f32, then u32 last so ncu_summary.json describes the headline).
# Run on the GPU box; results land in gpurun_out/profiles_out/ (copy into profiles/).
TAG=${1:-r02}
OUT=gpurun_out/profiles_out
mkdir -p $OUT
python bench.py > $OUT/${TAG}_bench_c2-u32-asc.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file /tmp/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-extras --no-cpu --no-e2e > /tmp/ncu_bench.log 2>&1
for w in u64-uniform:_u64 c2-f32-asc:_f32 c2-u32-asc:; do
  wl=${w%%:*}; suf=${w#*:}
  ncu --set full --import-source on --clock-control none -k regex:"k_scatter|k_final|k_hist|k_plan|k_sample" -c 20 \
    -f -o /tmp/prof_${TAG}$suf python tools/prof_sort.py --workload $wl --reps 1 > /tmp/ncu_$wl.log 2>&1
  python tools/make_profiles.py $TAG /tmp/launches_$TAG.csv /tmp/prof_${TAG}$suf.ncu-rep $wl > /dev/null
  cp profiles/${TAG}_ncu_full.md $OUT/${TAG}_ncu_full$suf.md
  for k in k_scatter k_final k_hist; do python tools/ncu_lines.py /tmp/prof_${TAG}$suf.ncu-rep $k 40 > $OUT/${TAG}_lines${suf}_$k.txt 2>&1; done
done
cp profiles/${TAG}_launches.md profiles/ncu_summary.json $OUT/
ls -la $OUT
