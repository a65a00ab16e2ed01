#!/bin/bash
# Alternating job-level A/B of runtime knobs (GPU box): value frames/s per run.
# usage: tools/ab_env.sh REPS "NAME=ENV..." "NAME=ENV..." ...   e.g. tools/ab_env.sh 2 "off=LB_ABUF=0" "on="
cd "$(dirname "$0")/.."
REPS=$1; shift
for r in $(seq $REPS); do
  for spec in "$@"; do
    name="${spec%%=*}"; envs="${spec#*=}"
    v=$(env $envs timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-configs --no-phases 2>/dev/null | tail -1 |
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'])")
    echo "$name $v"
  done
done
