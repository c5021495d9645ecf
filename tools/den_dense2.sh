# dense-cell share threshold for density rounds >= 1: the driver's C2 configuration and C4
out=gpurun_out/den_dense2.txt; : > $out
for fr in 0.5 0.6 0.65 0.7; do
  r=$(SPH_B200_DEN_DENSE=$fr timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'den', round(d['phase_ms']['density'],3), [round(x,3) for x in d['density_round_kernel_ms'][:3]])")
  echo "C2drv dense=$fr $r" >> $out
  r=$(SPH_B200_DEN_DENSE=$fr timeout 300 python bench.py --particles 16777216 --steps 5 --warmup 3 --e2e-steps 0 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'den', round(d['phase_ms']['density'],3), [round(x,3) for x in d['density_round_kernel_ms'][:3]])")
  echo "C4 dense=$fr $r" >> $out
done
cat $out
