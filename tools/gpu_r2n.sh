# r2n: no host sync in the rebin (round-0 item count read on the device): full GPU suite + timing
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2n.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2n.log
out=gpurun_out/r2n_bench.txt; : > $out
for N in 2097152 16777216; do for rep in 1 2; do
  r=$(timeout 300 python bench.py --particles $N --steps 5 --warmup 3 --e2e-steps 2 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), d['phase_ms'], [round(x,3) for x in d['density_round_kernel_ms'][:3]], 'e2e', round(d['e2e']['ms_per_step'],2), 'frac', round(d['roofline']['frac'],4))")
  echo "N=$N $r" >> $out
done; done
cat $out
