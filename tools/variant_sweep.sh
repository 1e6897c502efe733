#!/bin/bash
# same-box sweep of config-3 graph replay over the current tree and the variant copies given as args
for i in 1 2; do
  echo "== current"; python tools/level_sweep.py armor9k cc 6 | tail -1
  for d in "$@"; do echo "== $d"; (cd $d && python tools/level_sweep.py armor9k cc 6 | tail -1); done
done
