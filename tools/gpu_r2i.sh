# r2i: scheduling-invariance test, ncu of density round 0 (fixed selection), default bench line
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py -m gpu -x -q -k "scheduling" > gpurun_out/pytest_r2i.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2i.log
timeout 900 bash tools/profile.sh r2i
timeout 900 python bench.py > gpurun_out/bench_c2_r2i.json 2> gpurun_out/bench_c2_r2i.err
