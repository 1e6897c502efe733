#!/bin/bash
# build, GPU parity tests, level sweep, bench, ncu full capture of the CC level kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1 || { tail -30 gpurun_out/smoke.log; exit 1; }
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python tools/level_sweep.py armor9k cc 6 > gpurun_out/sweep.txt 2>&1; cat gpurun_out/sweep.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_cc_}" -c ${NCU_C:-18} -o gpurun_out/prof_cc -f python tools/prof_once.py 6 1 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
