#!/bin/bash
# Launch list + one full ncu capture of decode_kernel on the bench workload (run under gpurun).
# The capture runs the job as ONE launch (LB_NO_MIXED=1: under ncu's serialised
# replay the two concurrent mixed-width launches would not share the queue as
# they do live) on a quarter of the 4096-utterance job to bound the replay time;
# traffic is reported per utterance-frame and scaled to a bench launch.
# usage: tools/gpu_profile.sh <tag> [extra bench args]
tag=${1:-r02}; shift
mkdir -p gpurun_out
LB_NO_MIXED=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-configs --no-phases "$@" > gpurun_out/launches_${tag}.log 2>&1
LB_NO_MIXED=1 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 1 -c 1 \
    -o gpurun_out/prof_${tag} -f \
    python bench.py --utts 1024 --steps 1 --warmup 1 --no-e2e --no-cpu --no-configs --no-phases "$@" > gpurun_out/prof_${tag}.log 2>&1
echo "profile done: $(ls -la gpurun_out/prof_${tag}.ncu-rep 2>&1)"
