#!/bin/bash
# cmp_libs.sh under the driver's bench configuration (--steps 20 --warmup 5)
out=gpurun_out/cmp_libs_driver.txt; : > $out
for rep in $(seq ${REPS:-1}); do
for lib in paper_2502_16517_b200/lib/libsph_b200.so build/var_*/libsph_b200.so; do
  r=$(SPH_B200_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'den', round(d['phase_ms']['density'],3), [round(x,3) for x in d['density_round_kernel_ms'][:2]], 'for', round(d['phase_ms']['force'],3))")
  echo "$lib $r" >> $out
done; done
sort $out
