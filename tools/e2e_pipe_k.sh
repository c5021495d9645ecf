#!/bin/bash
# e2e (sph_step_host) time against the pipelined step's force chunk count (SPH_B200_PIPE_K).
# usage: BENCH_ARGS="--ic clustered" tools/e2e_pipe_k.sh 8 16
for k in "${@:-8 16}"; do
  r=$(SPH_B200_PIPE_K=$k timeout 300 python bench.py ${BENCH_ARGS:-} --steps 3 --warmup 3 --e2e-steps 6 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print(round(d['ms_per_step'],2), 'e2e', round(e['ms_per_step'],2), e['device_ms'])")
  echo "K=$k $r"
done
