#!/bin/bash
# same-box A/B of the current tree against _ab_old/ (a built copy of an older commit), graph replay
# of MESH SCHEME LEV (default config 3: armor9k cc 6), N rounds (default 3)
M=${MESH:-armor9k}; S=${SCHEME:-cc}; L=${LEV:-6}
for i in $(seq ${N:-3}); do
  echo -n "current "; python tools/level_sweep.py $M $S $L | tail -1
  echo -n "old     "; (cd _ab_old && python tools/level_sweep.py $M $S $L | tail -1)
done
