#!/bin/bash
# same-box A/B of an environment toggle on config-3 graph replay:  tools/ab_env.sh VAR=1 [VAR2=1 ...]
# (each arg is one variant's environment assignment; "-" = the default build)
for i in 1 2 3; do
  for v in - "$@"; do
    if [ "$v" = "-" ]; then echo -n "default   "; python tools/level_sweep.py armor9k cc 6 | tail -1
    else echo -n "$v "; env $v python tools/level_sweep.py armor9k cc 6 | tail -1; fi
  done
done
