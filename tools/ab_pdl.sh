timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 600 python bench.py > gpurun_out/bench_pdl.json 2> gpurun_out/bench_pdl.err
GG_PDL=0 timeout 600 python bench.py > gpurun_out/bench_nopdl.json 2> gpurun_out/bench_nopdl.err
for f in gpurun_out/bench_pdl.json gpurun_out/bench_nopdl.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['eager']['value'], d['e2e']['value'], d['roofline']['frac'], d['phases']['insert_ms_by_round'], d['phases']['grow_ms_per_step'], d['flatten']['gbs'], d['rw_config3']['ggarray_per_shard']['gbs'], d['rw_config3']['ggarray_global']['gbs'])"; done
tail -3 gpurun_out/bench_pdl.err
