#!/bin/bash
# Launch list + one full ncu capture of decode_kernel on the bench workload (run under gpurun).
# usage: tools/gpu_profile.sh <tag> [extra bench args]
tag=${1:-r01}; shift
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-configs "$@" > gpurun_out/launches_${tag}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 1 -c 1 \
    -o gpurun_out/prof_${tag} -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-configs "$@" > gpurun_out/prof_${tag}.log 2>&1
echo "profile done: $(ls -la gpurun_out/prof_${tag}.ncu-rep 2>&1)"
