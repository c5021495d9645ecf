# r2z: final validation of the round-2 state: full GPU suite, smoke, default bench, the
# driver's configuration, the reference arm (2 steps)
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2z.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2z.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2z.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_r2z.log
timeout 900 python bench.py > gpurun_out/bench_c2_r2z.json 2> gpurun_out/bench_c2_r2z.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_c2drv_r2z.json 2> gpurun_out/bench_c2drv_r2z.err
