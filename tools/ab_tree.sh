#!/bin/bash
# same-box A/B of the current tree against _ab_old/ (a built copy of an older commit), config-3
# graph replay, 3 rounds; then the timeline of both
for i in $(seq ${N:-3}); do
  echo -n "current "; python tools/level_sweep.py armor9k cc 6 | tail -1
  echo -n "old     "; (cd _ab_old && python tools/level_sweep.py armor9k cc 6 | tail -1)
done
