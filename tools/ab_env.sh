#!/bin/bash
# Dev (GPU): tools/mode_sweep.py under alternating environment settings,
# e.g. tools/ab_env.sh "VABFT_WAIT_NS=0" "VABFT_WAIT_NS=1000000"
for rep in 1 2; do
  for setting in "$@"; do
    env $setting timeout 300 python tools/mode_sweep.py 2>&1 | sed "s/^/[$setting] /"
  done
done
