#!/bin/bash
# The growarray-bench experiments on one B200 -> profiles/<round>_bench_cli/
# (then: python tools/summarize_cli.py profiles/<round>_bench_cli)
set -e
OUT=${1:-profiles/r02_bench_cli}
mkdir -p $OUT
CLI="python -m paper_2209_00103_b200.bench_cli"
for s in ggarray static doubling chunktable; do
  $CLI grow-insert-rw --structure $s --shards 512 --initial-size 1048576 --iterations 10 --algo scan \
      --work-passes 10 --repetitions 3 --out $OUT/grow_insert_rw_$s.csv
done
$CLI insert-algos --shards 32 --initial-size 1048576 --iterations 8 --work-passes 30 --repetitions 3 \
    --out $OUT/insert_algos.csv
$CLI shard-sweep --shards 1,8,64,512,4096 --initial-size 1048576 --iterations 6 --work-passes 5 --repetitions 2 --out $OUT/shard_sweep.csv
$CLI two-phase --shards 512 --initial-size 1048576 --iterations 6 --work-passes 10 --repetitions 3 \
    --out $OUT/two_phase.csv
$CLI memory-model --measure 3 --out $OUT/memory_model.csv
