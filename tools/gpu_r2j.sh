# r2j: ncu of density round 0 (mangled-name selection) + launch list
set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --cpu-baseline 0"
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "regex:density2_kernelILi20ELi1ELb0E" -s 3 -c 1 -o gpurun_out/density_r2j $B > gpurun_out/ncu_den_r2j.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:^force2_kernel -s 2 -c 1 \
    -o gpurun_out/force_r2j $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r2j.csv $B > gpurun_out/launches_r2j.log 2>&1
ls -la gpurun_out
