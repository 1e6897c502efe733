#!/bin/bash
# profiles for profiles/: ncu launch list of one refine (durations of every launch) and a full
# capture of the CC level kernels; plus the bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_once.py 6 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cc_" -c 18 -o gpurun_out/prof_cc -f python tools/prof_once.py 6 1 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
