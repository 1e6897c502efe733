#!/bin/bash
# quick GPU timing session: graph-replayed level sweeps (configs 3, 4, Loop torus) + config-5 frames
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1 || { tail -30 gpurun_out/smoke.log; exit 1; }
echo "== armor9k cc"; python tools/level_sweep.py armor9k cc 6
echo "== torus100k sqrt3"; python tools/level_sweep.py torus100k sqrt3 5
echo "== torus100k loop"; python tools/level_sweep.py torus100k loop 4
echo "== ico loop"; python tools/level_sweep.py ico loop 6 | tail -1
echo "== frames"; python tools/frames_once.py 4 16
