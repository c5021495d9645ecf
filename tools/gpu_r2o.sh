# r2o: round-2 evidence on the final kernels: benches C2 (+ cpu baseline), C3, C4, the C5 box on
# one GPU, the reference arm, and the ncu captures
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c2_r2o.json 2> gpurun_out/bench_c2_r2o.err
timeout 600 python bench.py --ic clustered --cpu-baseline 0 > gpurun_out/bench_c3_r2o.json 2> gpurun_out/bench_c3_r2o.err
timeout 900 python bench.py --particles 16777216 --cpu-baseline 0 --steps 5 > gpurun_out/bench_c4_r2o.json 2> gpurun_out/bench_c4_r2o.err
timeout 1500 python bench.py --particles 67108864 --cpu-baseline 0 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/bench_c5_r2o.json 2> gpurun_out/bench_c5_r2o.err
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r2o.json 2> gpurun_out/bench_ref_r2o.err
timeout 900 bash tools/profile.sh r2o
