#!/bin/bash
# Compare force variants with bench.py (one line per variant): lib x SPH_B200_FORCE2.
out=gpurun_out/cmp_force.txt; : > $out
run() { # name lib force2
  r=$(SPH_B200_LIB=$2 SPH_B200_FORCE2=$3 timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'den', d['phase_ms']['density'], d['density_round_kernel_ms'][:2], 'for', d['phase_ms']['force'], round(d['roofline']['frac'],4), round(d['roofline_density']['frac'],4))")
  echo "$1 $r" >> $out
}
run base_old paper_2502_16517_b200/lib/libsph_b200.so 0
run f2_m5 paper_2502_16517_b200/lib/libsph_b200.so 1
for lib in build/var_*/libsph_b200.so; do run $(basename $(dirname $lib)) $lib 1; done
cat $out
