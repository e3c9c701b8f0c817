#!/bin/bash
# Round-2 evidence run (one B200): bench line, reference arm, ncu launch list of
# one bench step, per-kernel metrics over every library kernel (prof_all.py),
# --set full of the hot kernels.  Summaries: tools/summarize_ncu.py,
# tools/summarize_all.py.
set -x
OUT=gpurun_out
mkdir -p $OUT
REP=/tmp/gg_prof
mkdir -p $REP
MET="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_op_atom.sum,lts__t_requests_op_red.sum,launch__registers_per_thread,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"
PROF_OUT=$OUT/plain timeout 300 python tools/prof_all.py > $OUT/prof_all_plain.log 2>&1
if [ -z "$SKIP_BENCH" ]; then
  timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
  timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 3 --quick --no-cpu > $OUT/bench_ncu.log 2>&1
timeout 1200 ncu --nvtx --nvtx-include "profiled/" --metrics $MET --clock-control none \
    -k regex:"^(k_|spin_kernel)" --csv --log-file $OUT/prof_all.csv \
    python tools/prof_all.py > $OUT/prof_all.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "profiled/" \
    -k regex:"k_walk|k_rw_global" -o $REP/prof_full -f python tools/prof_target.py > $OUT/prof.log 2>&1
ncu -i $REP/prof_full.ncu-rep --page raw --csv > $OUT/prof_raw.csv 2>/dev/null
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "profiled/" \
    -k regex:"^(k_walk_shard|k_lanes_chunk|k_push_if|k_flat_insert_block|k_flat_append|k_gather)" \
    -o $REP/prof_paths_full -f python tools/prof_all.py > $OUT/prof_paths.log 2>&1
ncu -i $REP/prof_paths_full.ncu-rep --page raw --csv > $OUT/prof_paths_raw.csv 2>/dev/null
ncu -i $REP/prof_full.ncu-rep --page details --csv > $OUT/prof_details.csv 2>/dev/null
ncu -i $REP/prof_paths_full.ncu-rep --page details --csv > $OUT/prof_paths_details.csv 2>/dev/null
ls -la $OUT $REP
du -sh $OUT
