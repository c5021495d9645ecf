# r2s: ncu of the density round-1 kernels late in the driver's run (step ~15 of 25)
set -x
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 5 --e2e-steps 0 --cpu-baseline 0"
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "regex:density2_kernelILi20ELi4ELb0E" -s 28 -c 1 -o gpurun_out/den_r1sparse_r2s $B > gpurun_out/ncu_r2s_a.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "regex:density2_kernelILi20ELi1ELb0E" -s 43 -c 2 -o gpurun_out/den_r1dense_r2s $B > gpurun_out/ncu_r2s_b.log 2>&1
