#!/bin/bash
# quick GPU session: build, smoke, level sweep, bench (no tests, no ncu)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1 || { tail -30 gpurun_out/smoke.log; exit 1; }
python tools/level_sweep.py armor9k cc 6 > gpurun_out/sweep.txt 2>&1; cat gpurun_out/sweep.txt
python tools/level_sweep.py torus100k sqrt3 5 > gpurun_out/sweep_s3.txt 2>&1; cat gpurun_out/sweep_s3.txt
python tools/level_sweep.py ico loop 6 > gpurun_out/sweep_loop.txt 2>&1; cat gpurun_out/sweep_loop.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
