#!/bin/bash
# Per-config ncu metrics of each config's dominant kernel (one launch each, cold cache, clocks unlocked).
# Usage (on the GPU box): bash tools/ncu_configs.sh gpurun_out/prof
out=${1:-gpurun_out/prof}; mkdir -p "$out"
M=gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,launch__grid_size,launch__block_size,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,smsp__warp_issue_stalled_wait_per_warp_active.pct,smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct
run() {  # name, kernel regex, quick_time args
  timeout 600 ncu --metrics $M --clock-control none -k regex:"$2" -c 1 --csv --log-file "$out/ncu_$1.csv" python tools/quick_time.py $3 > /dev/null 2>&1
}
run c1-10k k_reg32b "C1-10k"
run c2-full k_reg16c "C2-full"
run c3 k_blocked_reg "C3"
run c4 k_creg32 "C4"
run c5 k_blocked_reg "C5"
# C4 on the QR route: the two QR kernels (quick_time has no qr config; use the probe)
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_qr_col|k_applyq_col" -c 2 --csv --log-file "$out/ncu_c4-qr.csv" python tools/qr_route_probe.py > /dev/null 2>&1
