# r2h: ncu of the round-2 kernels, sanitizer on the persistent sweeps, persistent A/B on one box
set -x
mkdir -p gpurun_out
timeout 900 bash tools/profile.sh r2h
for t in memcheck racecheck synccheck; do
  SAN_N=131072 SAN_PPC=64 timeout 900 compute-sanitizer --tool $t python tools/sanitize.py > gpurun_out/san_$t.txt 2>&1
done
out=gpurun_out/persist_ab.txt; : > $out
for rep in 1 2 3; do for v in "0 0" "1 1"; do set -- $v
  r=$(SPH_B200_PERSIST0=$1 SPH_B200_F2_PERSIST=$2 timeout 300 python bench.py --steps 6 --warmup 3 --e2e-steps 0 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'den', round(d['phase_ms']['density'],3), [round(x,3) for x in d['density_round_kernel_ms'][:2]], 'for', round(d['phase_ms']['force'],3))")
  echo "persist0=$1 f2persist=$2 $r" >> $out
done; done
cat $out
