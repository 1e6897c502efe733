#!/bin/bash
# same-box A/B: graph-replayed config-3 level sweep with the current library and with _ab_old/
for i in 1 2; do
  echo "== current"; python tools/level_sweep.py armor9k cc 6 | tail -2
  echo "== old"; (cd _ab_old && python tools/level_sweep.py armor9k cc 6 | tail -2)
done
