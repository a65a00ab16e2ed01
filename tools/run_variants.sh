#!/bin/bash
# Per-phase timing of each variant built by tools/variants.sh (GPU box).
# usage: tools/run_variants.sh U T name1 name2 ...
cd "$(dirname "$0")/.."
U=$1; T=$2; shift 2
for name in "$@"; do
  echo "== $name"
  LB_SO_PATH=build/variants/$name.so timeout 300 python tools/phases.py $U $T ${CFG:-2x640} 2>&1 | tail -3
done
