#!/bin/bash
# Compare runtime variants (environment settings) with bench.py, one line per variant.
# usage: tools/cmp_env.sh "NAME:ENV=V ENV2=V" ...
out=gpurun_out/cmp_env.txt; : > $out
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  r=$(env $envs timeout 300 python bench.py ${BENCH_ARGS:-} --steps 5 --warmup 3 --e2e-steps 0 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'rebin', d['phase_ms']['rebin'], 'den', round(d['phase_ms']['density'],3), [round(x,3) for x in d['density_round_kernel_ms'][:3]], 'for', round(d['phase_ms']['force'],3), 'frac', round(d['roofline']['frac'],4), round(d['roofline_density']['frac'],4))")
  echo "$name $r" >> $out
done
cat $out
