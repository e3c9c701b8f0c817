#!/bin/bash
# Evidence run for profiles/: bench line, ncu launch list of one bench step,
# ncu --set full of the dominant kernel (duplicate insert, last round) + r/w + flatten.
set -x
OUT=gpurun_out
python bench.py > $OUT/bench.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 3 --quick --no-cpu > $OUT/bench_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_walk|k_rw_global" -s 10 -c 5 \
    -o $OUT/prof_full python tools/prof_target.py > $OUT/prof.log 2>&1
ncu -i $OUT/prof_full.ncu-rep --page raw --csv > $OUT/prof_raw.csv 2>/dev/null
ncu -i $OUT/prof_full.ncu-rep --page details --csv > $OUT/prof_details.csv 2>/dev/null
# L2 atomic traffic of the atomic-bound kernels (static insert per element / warp / block,
# device push_back warp / block, per-lane-count insert)
ncu --metrics "regex:^lts__t_(requests|sectors)_op_(atom|red)\.sum$,gpu__time_duration.sum" --clock-control none \
    --csv --log-file $OUT/atomics.csv -k regex:"k_flat_insert|k_push_if|k_lanes_insert" \
    python tools/prof_atomics.py > $OUT/atomics.log 2>&1
