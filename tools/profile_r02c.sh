#!/bin/bash
# Round-2 final captures after the launch-shape tuning (2 / 3 CTAs per SM): ncu --set full of the
# decode kernel on configs 2/3/4, range64 through the access layout, and the bench launch list.
# Outputs land in gpurun_out/r02c/.
set -u
O=gpurun_out/r02c
mkdir -p $O
NCU="ncu --set full --import-source on --clock-control none"
for c in 2 3 4; do
  $NCU -k regex:lc_decode_kernel -c 1 -o $O/decode_c$c python tools/prof_decode.py --config $c --reps 1 > $O/decode_c$c.log 2>&1
done
$NCU -k regex:lc_range64 -c 1 -o $O/range64_dir python tools/prof_access.py --reps 1 --only layout > $O/range64_dir.log 2>&1
$NCU -k regex:"lc_union|lc_decode_kernel|lc_isect" -c 12 -o $O/union python tools/prof_union.py > $O/union.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu > $O/launches_bench.log 2>&1
# summaries on the box (gpurun_out/ travels back only below 64 MiB: the union report is dropped)
python tools/ncu_summary.py $O/union.ncu-rep --out $O/union_full.txt > /dev/null 2>&1
rm -f $O/union.ncu-rep
ls -la $O
