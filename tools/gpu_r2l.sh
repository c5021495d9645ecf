# r2l: randomised parity sweep on the round-2 kernels + a 2-rank decomposed bench (ranks share
# the one GPU, gloo transport) and a clustered 2-rank one
set -x
mkdir -p gpurun_out
timeout 1500 python tools/parity_sweep.py --configs 120 --seed 2027 --out gpurun_out/parity_sweep_r2.md > gpurun_out/parity_sweep_r2.log 2>&1
SPH_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --particles 1048576 > gpurun_out/bench_2rank_r2.json 2> gpurun_out/bench_2rank_r2.err
SPH_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 3 --warmup 3 --particles 1048576 --ic clustered > gpurun_out/bench_2rank_c3_r2.json 2> gpurun_out/bench_2rank_c3_r2.err
