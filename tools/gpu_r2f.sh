# r2f: full GPU suite + benches C2/C3/C4 on the current defaults
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2f.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2f.log
timeout 900 python bench.py > gpurun_out/bench_c2_r2f.json 2> gpurun_out/bench_c2_r2f.err
timeout 600 python bench.py --ic clustered --cpu-baseline 0 > gpurun_out/bench_c3_r2f.json 2> gpurun_out/bench_c3_r2f.err
timeout 600 python bench.py --particles 16777216 --cpu-baseline 0 --steps 5 > gpurun_out/bench_c4_r2f.json 2> gpurun_out/bench_c4_r2f.err
