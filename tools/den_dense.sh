# density rounds >= 1: dense-cell rule (share SPH_B200_DEN_DENSE, count SPH_B200_DEN_DENSE_ABS)
# and lanes per sparse particle (SPH_B200_DEN_JS1) on C2, C3 (clustered), C4
out=gpurun_out/den_dense.txt; : > $out
for cfg in "2097152 uniform" "2097152 clustered" "16777216 uniform"; do set -- $cfg; N=$1; IC=$2
for v in "4 0.5 1000000000" "4 0.5 512" "4 0.5 256" "4 0.5 1024" "2 0.35 1000000000" "2 0.35 512"; do set -- $v
  r=$(SPH_B200_DEN_JS1=$1 SPH_B200_DEN_DENSE=$2 SPH_B200_DEN_DENSE_ABS=$3 timeout 300 python bench.py --particles $N --ic $IC --steps 5 --warmup 3 --e2e-steps 0 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'den', round(d['phase_ms']['density'],3), [round(x,3) for x in d['density_round_kernel_ms'][:3]], 'for', round(d['phase_ms']['force'],3))")
  echo "N=$N ic=$IC js1=$1 dense=$2 abs=$3 $r" >> $out
done; done
cat $out
