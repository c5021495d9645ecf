#!/bin/bash
# ncu evidence for profiles/: launch list of a short bench run + one full capture of each
# hot kernel. Run under gpurun (one GPU). Outputs into gpurun_out/.
set -x
TAG=${1:-r1}
B="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --cpu-baseline 0"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/launches_$TAG.log 2>&1
# one launch of each pair sweep after the IC and the warm-up step (steady state)
ncu --set full --clock-control none --import-source on -k regex:^force2_kernel -s 2 -c 1 \
    -o gpurun_out/force_$TAG $B > /dev/null 2>&1
# density round 0 of the second step: the first density2_kernel<20, 1, 0> launch of each
# step is round 0 (then the dense-cell launches of rounds 1 and 2 follow under the same name)
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "regex:density2_kernelILi20ELi1ELb0E" -s 3 -c 1 \
    -o gpurun_out/density_$TAG $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"^kick2_kernel|^drift_kernel|^kick1_kernel" -s 3 -c 3 -o gpurun_out/linear_$TAG $B > /dev/null 2>&1
ls -la gpurun_out
