# density round-0 lanes per particle (SPH_B200_DEN_JS0) at C2 and C4
out=gpurun_out/den_js.txt; : > $out
for N in 2097152 16777216; do for js in 1 2 4; do
  r=$(SPH_B200_DEN_JS0=$js timeout 300 python bench.py --particles $N --steps 4 --warmup 3 --e2e-steps 0 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'den', round(d['phase_ms']['density'],3), [round(x,3) for x in d['density_round_kernel_ms'][:3]], 'for', round(d['phase_ms']['force'],3))")
  echo "N=$N js0=$js $r" >> $out
done; done
cat $out
