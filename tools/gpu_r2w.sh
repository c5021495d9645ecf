# r2w: final round-2 state: full GPU suite, benches (default C2 with CPU baseline, the driver's
# 20+5-step C2, C3, C4), ncu captures
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2w.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2w.log
timeout 900 python bench.py > gpurun_out/bench_c2_r2w.json 2> gpurun_out/bench_c2_r2w.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --cpu-baseline 0 > gpurun_out/bench_c2drv_r2w.json 2> gpurun_out/bench_c2drv_r2w.err
timeout 600 python bench.py --ic clustered --cpu-baseline 0 > gpurun_out/bench_c3_r2w.json 2> gpurun_out/bench_c3_r2w.err
timeout 900 python bench.py --particles 16777216 --cpu-baseline 0 --steps 5 > gpurun_out/bench_c4_r2w.json 2> gpurun_out/bench_c4_r2w.err
timeout 900 bash tools/profile.sh r2w
