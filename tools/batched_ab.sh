#!/bin/bash
# batched-mode frames/s at several batch sizes for the variants built by tools/variants.sh
cd "$(dirname "$0")/.."
for name in "$@"; do
  for U in 1 8 32; do
    echo "$name U=$U: $(LB_SO_PATH=build/variants/$name.so python tools/phases_batched.py $U 300 2>&1 | tail -1)"
  done
done
