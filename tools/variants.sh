#!/bin/bash
# Build compile-time variants of liblatbeam_b200.so into build/variants/<name>.so
# usage: tools/variants.sh name1:"-DFOO=1 -DBAR" name2:"..."   (then LB_SO_PATH=... python tools/phases.py)
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
pids=()
for spec in "$@"; do
  name="${spec%%:*}"; defs="${spec#*:}"
  /usr/local/cuda/bin/nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -std=c++17 -fmad=false \
    -Xcompiler -fPIC,-O2 -Xptxas -v $defs -shared -o build/variants/$name.so \
    paper_1804_03243_b200/csrc/latbeam_b200.cu -lcudart 2> build/variants/$name.ptxas.txt &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
for spec in "$@"; do
  name="${spec%%:*}"
  echo "$name: $(grep -A2 'decode_kernelILi640ELi.ELb0ELb0' build/variants/$name.ptxas.txt | grep -o '[0-9]* bytes spill stores, [0-9]* bytes spill loads' | head -1)"
done
