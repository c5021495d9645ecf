# r2c: device-counted density rounds: parity subset + C2/C4 timing with and without
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py tests/test_decomp.py -m gpu -x -q > gpurun_out/pytest_r2c.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2c.log
out=gpurun_out/devrounds.txt; : > $out
for N in 2097152 16777216; do for dr in 0 1 0 1; do
  r=$(SPH_B200_DEV_ROUNDS=$dr timeout 300 python bench.py --particles $N --steps 5 --warmup 3 --e2e-steps 0 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'den', round(d['phase_ms']['density'],3), [round(x,3) for x in d['density_round_kernel_ms'][:3]], 'for', round(d['phase_ms']['force'],3), 'launches', d['gpu_launches_per_step'])")
  echo "N=$N dev_rounds=$dr $r" >> $out
done; done
cat $out
