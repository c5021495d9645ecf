#!/bin/bash
# Time the pair kernels of each variant build (build/var_*/libsph_b200.so) with bench.py.
out=gpurun_out/variants.txt; : > $out
for lib in paper_2502_16517_b200/lib/libsph_b200.so build/var_*/libsph_b200.so; do
  r=$(SPH_B200_LIB=$lib python bench.py --steps 3 --warmup 2 --e2e-steps 0 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), d['phase_ms']['density'], d['phase_ms']['force'])")
  echo "$lib $r" >> $out
done
cat $out
