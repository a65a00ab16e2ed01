#!/bin/bash
# CTA size / emit batch width sweep of the lane kernel (build/variants/extra.so, -DLB_EXTRA)
cd "$(dirname "$0")/.."
export LB_SO_PATH=build/variants/extra.so
for spec in ${SPECS:-768:2 704:2 672:2 640:1 640:2 608:2 576:2 576:3}; do
  t=${spec%%:*}; u=${spec##*:}
  echo "threads=$t unr=$u: $(LB_UNR=$u timeout 300 python tools/phases.py ${1:-64} ${2:-100} 2x$t 2>&1 | head -1)"
done
