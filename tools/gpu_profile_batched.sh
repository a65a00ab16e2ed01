#!/bin/bash
# Launch list + one full ncu capture of the batched-mode phase kernels (C2: one utterance).
tag=${1:-r01}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_batched_${tag}.csv \
    python tools/phases_batched.py 1 60 > gpurun_out/launches_batched_${tag}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:b_winners -s 40 -c 1 \
    -o gpurun_out/prof_batched_${tag} -f python tools/phases_batched.py 1 60 > gpurun_out/prof_batched_${tag}.log 2>&1
echo "done $(ls gpurun_out/prof_batched_${tag}.ncu-rep)"
