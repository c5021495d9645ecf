# r2ab: sanitizer on the tail-map rebin + final benches (default, driver configuration, C3, C4)
set -x
mkdir -p gpurun_out
for t in memcheck racecheck; do
  SAN_N=131072 SAN_PPC=64 timeout 900 compute-sanitizer --tool $t python tools/sanitize.py > gpurun_out/san2_$t.txt 2>&1
done
timeout 900 python bench.py > gpurun_out/bench_c2_r2ab.json 2> gpurun_out/bench_c2_r2ab.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --cpu-baseline 0 > gpurun_out/bench_c2drv_r2ab.json 2> gpurun_out/bench_c2drv_r2ab.err
timeout 600 python bench.py --ic clustered --cpu-baseline 0 > gpurun_out/bench_c3_r2ab.json 2> gpurun_out/bench_c3_r2ab.err
timeout 900 python bench.py --particles 16777216 --cpu-baseline 0 --steps 5 > gpurun_out/bench_c4_r2ab.json 2> gpurun_out/bench_c4_r2ab.err
