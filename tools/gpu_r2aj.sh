#!/bin/bash
# r2aj: the C5w weak-scaling N=1 point (8,479,744 particles, nx = 91) and a final GPU suite.
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --particles 8479744 --steps 5 --warmup 3 --cpu-baseline 0 \
  > gpurun_out/r2aj_bench_c5w_n1.json 2> gpurun_out/r2aj_bench_c5w_n1.err
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2aj_pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2aj_smoke.log 2>&1
