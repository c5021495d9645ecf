set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r2a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2a.log
timeout 600 python bench.py > gpurun_out/bench_c2_r2a.json 2> gpurun_out/bench_c2_r2a.err
timeout 600 python bench.py --ic clustered --cpu-baseline 0 > gpurun_out/bench_c3_r2a.json 2> gpurun_out/bench_c3_r2a.err
timeout 600 python bench.py --particles 16777216 --cpu-baseline 0 --steps 5 > gpurun_out/bench_c4_r2a.json 2> gpurun_out/bench_c4_r2a.err
timeout 900 bash tools/profile.sh r2a
