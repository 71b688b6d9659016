#!/bin/bash
# Round-2 (late) captures: corpus batch decode, the fused union's kernels, range64 (ncu --set
# full with source), for tools/ncu_sass.py.  Outputs land in gpurun_out/r02b/.
set -u
O=gpurun_out/r02b
mkdir -p $O
NCU="ncu --set full --import-source on --clock-control none"
$NCU -k regex:lc_decode_batch -c 1 -o $O/batch python tools/prof_batch.py --reps 1 --per-list 1 > $O/batch.log 2>&1
$NCU -k regex:"lc_union|lc_decode_kernel|lc_scan|lc_place|lc_compact" -c 12 -o $O/union python tools/prof_union.py > $O/union.log 2>&1
$NCU -k regex:lc_range64 -c 1 -o $O/range64 python tools/prof_access.py --reps 1 --only plain > $O/range64.log 2>&1
ls -la $O
