#!/bin/bash
# small-level latency study: graph increments per level, live probes of levels -1..3, ncu full
# capture (with source) of every kernel of one eager config-3 refine
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/level_sweep.py armor9k cc 6 > gpurun_out/sweep.txt 2>&1; cat gpurun_out/sweep.txt
for l in -1 0 1 2 3 4; do python tools/probe_level.py $l; done > gpurun_out/probe_small.txt 2>&1; cat gpurun_out/probe_small.txt
timeout 900 ncu --set full --clock-control none --import-source on -c 60 -o gpurun_out/prof_small -f python tools/prof_once.py 6 1 > gpurun_out/ncu_small.log 2>&1
tail -3 gpurun_out/ncu_small.log
