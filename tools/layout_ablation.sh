#!/bin/bash
# BASELINE config 4: layout ablation (AoS in place / convert per call / resident SoA) at
# n = 2^24, ppc = 1024. Times one full step per layout and captures per-kernel DRAM traffic
# and pipe utilisation with ncu. Run under gpurun (1 GPU). Outputs in gpurun_out/.
N=${N:-16777216}
for L in resident aos convert; do
  python bench.py --particles $N --layout $L --steps 3 --warmup 2 --e2e-steps 0 --cpu-baseline 0 \
      > gpurun_out/abl_$L.json 2> gpurun_out/abl_$L.err
  ncu --clock-control none \
      -k regex:"force2_kernel|density2_kernel|drift_kernel|kick1_kernel|kick2_kernel|gather_kernel|scatter_kernel|jview_|permute_fused|chunk_box" \
      -c 16 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,lts__t_bytes.sum \
      --csv --log-file gpurun_out/abl_ncu_$L.csv \
      python bench.py --particles $N --layout $L --steps 1 --warmup 1 --e2e-steps 0 --cpu-baseline 0 > /dev/null 2>&1
done
ls -la gpurun_out/abl_*
