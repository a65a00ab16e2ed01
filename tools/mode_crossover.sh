#!/bin/bash
# batched vs persistent-lane frames/s by batch size (C2 graph, costs in HBM)
cd "$(dirname "$0")/.."
for U in ${US:-16 32 40 48 56 64}; do
  echo "U=$U batched: $(LB_MODE=batched python tools/phases_batched.py $U 300 2>&1 | tail -1)   lane: $(LB_MODE=lane python tools/phases_batched.py $U 300 2>&1 | tail -1)"
done
