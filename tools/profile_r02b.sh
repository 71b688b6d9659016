#!/bin/bash
# Round-2 (late) captures on one B200, final build: corpus batch decode, the fused union's
# kernels, range64 through the access layout (ncu --set full with source, for
# tools/ncu_summary.py / tools/ncu_sass.py) and the launch list of the bench command.
# Outputs land in gpurun_out/r02b/.
set -u
O=gpurun_out/r02b
mkdir -p $O
NCU="ncu --set full --import-source on --clock-control none"
$NCU -k regex:lc_decode_batch -c 1 -o $O/batch python tools/prof_batch.py --reps 1 --per-list 1 > $O/batch.log 2>&1
$NCU -k regex:"lc_union|lc_decode_kernel|lc_isect" -c 12 -o $O/union python tools/prof_union.py > $O/union.log 2>&1
$NCU -k regex:lc_range64 -c 1 -o $O/range64_dir python tools/prof_access.py --reps 1 --only layout > $O/range64_dir.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu > $O/launches_bench.log 2>&1
ls -la $O
