#!/bin/bash
# frames/s of the automatic mode choice by batch size (C2 graph, costs in HBM)
cd "$(dirname "$0")/.."
for U in ${US:-1 4 5 8 12 15 16 17 20 24 28 32 33 36 40 44 48 64}; do
  echo "U=$U auto: $(LB_MODE_DEBUG=1 python tools/phases_batched.py $U 300 2>&1 | grep -E 'mode|frames' | tail -2 | tr '\n' ' ')"
done
