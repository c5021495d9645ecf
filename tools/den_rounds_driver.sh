# density rounds >= 1 under the driver's bench configuration (--steps 20 --warmup 5: pending
# particles grow from ~2 % to ~60 % over the run): lanes per sparse particle x dense threshold
out=gpurun_out/den_rounds_driver.txt; : > $out
for v in "4 0.5" "4 0.35" "4 0.7" "2 0.5" "2 0.7" "4 0.9" "2 0.35" "1 0.0"; do set -- $v
  r=$(SPH_B200_DEN_JS1=$1 SPH_B200_DEN_DENSE=$2 timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'den', round(d['phase_ms']['density'],3), [round(x,3) for x in d['density_round_kernel_ms'][:3]], 'for', round(d['phase_ms']['force'],3))")
  echo "js1=$1 dense=$2 $r" >> $out
done
cat $out
