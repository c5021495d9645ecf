# density rounds >= 1: lanes per particle (SPH_B200_DEN_JS1) and dense-cell threshold
out=gpurun_out/den_js1.txt; : > $out
for N in 2097152 16777216; do for v in "4 0.5" "4 0.65" "4 0.8" "8 0.5" "8 0.65" "8 0.8" "8 1.01" "2 0.35"; do set -- $v
  r=$(SPH_B200_DEN_JS1=$1 SPH_B200_DEN_DENSE=$2 timeout 300 python bench.py --particles $N --steps 5 --warmup 3 --e2e-steps 0 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'den', round(d['phase_ms']['density'],3), [round(x,3) for x in d['density_round_kernel_ms'][:3]], 'for', round(d['phase_ms']['force'],3))")
  echo "N=$N js1=$1 dense=$2 $r" >> $out
done; done
cat $out
