#!/bin/bash
# e2e (sph_step_host) time against the pipelined step's force chunk count (SPH_B200_PIPE_K)
# and shrinking tail (SPH_B200_PIPE_TAIL). usage: BENCH_ARGS="--ic clustered" tools/e2e_pipe_k.sh "16 2" "24 3"
out=gpurun_out/e2e_pipe_k.txt; : > $out
for kt in "${@:-16 2}"; do set -- $kt
  r=$(SPH_B200_PIPE_K=$1 SPH_B200_PIPE_TAIL=${2:-2} timeout 300 python bench.py ${BENCH_ARGS:-} --steps 3 --warmup 3 --e2e-steps 6 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print(round(d['ms_per_step'],2), 'e2e', round(e['ms_per_step'],2), e['device_ms'])")
  echo "K=$1 T=${2:-2} $r" | tee -a $out
done
