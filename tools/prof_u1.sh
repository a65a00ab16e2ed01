#!/bin/bash
# ncu --set full of one decode_kernel launch at U lanes (default 1), T frames: intrinsic per-lane latency.
U=${1:-1}; T=${2:-30}; tag=${3:-u1}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 1 -c 1 -o gpurun_out/prof_${tag} -f \
    python tools/phases.py $U $T ${CONF:-2x768} > gpurun_out/prof_${tag}.log 2>&1
echo "done $(ls -la gpurun_out/prof_${tag}.ncu-rep)"
