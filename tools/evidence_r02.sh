#!/bin/bash
# Full round-2 evidence run on one B200: GPU tests, smoke, the ncu / bench
# evidence (tools/profile_r02.sh), the growarray-bench CLI suite, and the
# per-path probes (push_if / lanes throughput, host time per call, VMM cost).
OUT=gpurun_out
mkdir -p $OUT $OUT/probes
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/gputest.log 2>&1; echo "rc=$?" >> $OUT/gputest.log
timeout 300 python tools/cold_probe.py > $OUT/cold_probe.json 2>&1
bash tools/profile_r02.sh > $OUT/profile_r02.log 2>&1
for p in push_if_probe lanes_probe lanes_host_probe ragged_host_probe view_cost_probe gather_probe vmm_fresh_probe; do
  timeout 400 python tools/$p.py > $OUT/probes/$p.json 2> $OUT/probes/$p.err
done
timeout 1200 bash tools/run_cli_suite.sh $OUT/bench_cli > $OUT/cli.log 2>&1
tail -n 2 $OUT/gputest.log
