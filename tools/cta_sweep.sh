#!/bin/bash
# Lane CTA-size sweep of the decode kernel on the C4 shape (run under gpurun).
# The in-tree build carries the 512/640/768-thread variants; the wider sweep in
# DESIGN.md §10 (384..768 threads, UNR 1..4) used extra template instantiations
# that were removed after 640 won.
# usage: tools/cta_sweep.sh [U] [T]
cd "$(dirname "$0")/.."
for t in ${THREADS:-768 640 512}; do
  echo "threads=$t: $(timeout 300 python tools/phases.py ${1:-64} ${2:-100} 2x$t 2>&1 | head -1)"
done
