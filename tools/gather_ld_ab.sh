#!/bin/bash
# A/B of the random element read's cache policy in k_gather (GG_GATHER_LD,
# see ld_rand in gg_device.cuh): get_many / set_many timing (gather_probe.py)
# and the L2 sectors / DRAM bytes the gather requests under ncu, per mode.
OUT=${1:-gpurun_out/gather_ld}
mkdir -p $OUT
for m in 0 1 2 3 4; do
  GG_GATHER_LD=$m timeout 300 python tools/gather_probe.py > $OUT/probe_$m.json 2> $OUT/probe_$m.err
  GG_PROBE_ONE=0 GG_GATHER_LD=$m timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum \
    --clock-control none -k regex:k_gather --csv --log-file $OUT/ncu_$m.csv python tools/l2fetch_probe.py > $OUT/ncu_$m.log 2>&1
done
