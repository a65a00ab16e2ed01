#!/bin/bash
cd /root/repo
for r in 1 2; do
for spec in "t4=" "t2=LB_STAGE_THREADS=2" "t6=LB_STAGE_THREADS=6" "t8=LB_STAGE_THREADS=8" "r256=LB_RING_SLOTS=256"; do
  name="${spec%%=*}"; envs="${spec#*=}"
  v=$(env $envs timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-configs --no-phases 2>/dev/null | tail -1 |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']))")
  echo "$name $v"
done; done
