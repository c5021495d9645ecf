# r2b: parity of the operand-cost rewrites (default build) + timing of the variants
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py -m gpu -x -q -k "fast or symmetric or isolated or edge or deterministic or pipelined" > gpurun_out/pytest_r2b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2b.log
STEPS=6 timeout 1200 bash tools/cmp_libs.sh
