#!/bin/bash
# quick bench sweep: prints value, ms/step, roofline frac, kernel ms
for a in "$@"; do
  out=$(timeout 600 python bench.py --steps 3 --warmup 1 --no-cpu --no-e2e --no-configs $a 2>/dev/null | tail -1)
  echo "$a => $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],1), round(d["roofline"]["frac"],4), round(d["roofline"]["kernel_ms_per_launch"],1))' 2>&1)"
done
