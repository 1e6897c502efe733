#!/bin/bash
# one GPU session: build, parity tests, bench (N=1, incl. the frames job), bench --config 5, ncu
# launch list of config 3, ncu full capture of the final-level CC kernels and of the blocked SpMM
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1 || { tail -30 gpurun_out/smoke.log; exit 1; }
timeout 900 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
timeout 600 python bench.py --config 5 > gpurun_out/bench5.json 2>> gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_once.py 6 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cc_|k_crease" -c 40 -o gpurun_out/prof_cc -f python tools/prof_once.py 6 1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rb_eval" -s 1 -c 1 -o gpurun_out/prof_rb -f python tools/rm_once.py > gpurun_out/ncu_rb.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_rb.csv python tools/rm_once.py > /dev/null 2>&1
fi
ls -la gpurun_out
