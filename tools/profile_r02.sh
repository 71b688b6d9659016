#!/bin/bash
# Round-2 evidence capture on one B200 (run through gpurun from the repo root):
#   ncu --set full of the final decode kernel on configs 2/3/4, of the access-layout kernels,
#   of range64 and of the corpus batch decode; the launch list of the bench command; the
#   random-gather ceiling microbenchmark.  Outputs land in gpurun_out/r02/.
set -u
O=gpurun_out/r02
mkdir -p $O
NCU="ncu --set full --import-source on --clock-control none"
for c in 2 3 4; do
  $NCU -k regex:lc_decode_kernel -c 1 -o $O/decode_c$c python tools/prof_decode.py --config $c --reps 1 > $O/decode_c$c.log 2>&1
done
$NCU -k regex:lc_access_dir -c 2 -o $O/access_dir python tools/prof_access.py --reps 1 --only layout > $O/access_dir.log 2>&1
$NCU -k regex:lc_access_kernel -c 1 -o $O/access_plain python tools/prof_access.py --reps 1 --only plain > $O/access_plain.log 2>&1
$NCU -k regex:lc_decode_batch -c 1 -o $O/batch python tools/prof_batch.py --reps 1 --per-list 1 > $O/batch.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/gather_pattern tools/gather_pattern.cu
./build/gather_pattern > $O/gather_pattern.txt 2>&1
ncu --metrics dram__sectors_read.sum,gpu__time_duration.sum --clock-control none --csv ./build/gather_pattern > $O/gather_pattern_ncu.csv 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu > $O/launches_bench.log 2>&1
ls -la $O
