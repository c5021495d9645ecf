# r2d: persistent round-0 density / persistent force2: parity with both on + timing
set -x
mkdir -p gpurun_out
SPH_B200_PERSIST0=1 SPH_B200_F2_PERSIST=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py -m gpu -x -q -k "fast or symmetric or isolated or edge or deterministic or pipelined or nonconvergence" > gpurun_out/pytest_r2d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2d.log
out=gpurun_out/persist.txt; : > $out
for N in 2097152 16777216; do for v in "0 0" "1 0" "0 1" "1 1" "0 0" "1 1"; do set -- $v
  r=$(SPH_B200_PERSIST0=$1 SPH_B200_F2_PERSIST=$2 timeout 300 python bench.py --particles $N --steps 5 --warmup 3 --e2e-steps 2 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'den', round(d['phase_ms']['density'],3), [round(x,3) for x in d['density_round_kernel_ms'][:3]], 'for', round(d['phase_ms']['force'],3), 'e2e', round(d['e2e']['ms_per_step'],2))")
  echo "N=$N persist0=$1 f2persist=$2 $r" >> $out
done; done
cat $out
