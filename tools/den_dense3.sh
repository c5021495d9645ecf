# dense threshold 0.5 vs 0.9 under 20+5-step runs at C2 and C4
out=gpurun_out/den_dense3.txt; : > $out
for N in 2097152 16777216; do for fr in 0.5 0.9; do
  r=$(SPH_B200_DEN_DENSE=$fr timeout 900 python bench.py --particles $N --steps 20 --warmup 5 --e2e-steps 0 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'den', round(d['phase_ms']['density'],3), [round(x,3) for x in d['density_round_kernel_ms'][:3]])")
  echo "N=$N 20+5 dense=$fr $r" >> $out
done; done
cat $out
