#!/bin/bash
# ncu counters of the blocked-layer kernels across T_b and modes (cfg2), one
# launch each: time, DRAM and L2 bytes, FMA-pipe and tensor-pipe activity.
# Every command is first run plainly (must exit 0) before it is profiled.
set -e
OUT=${1:-gpurun_out/ncu_sweep}
mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum
for mode in f32 bf16 tf32; do
  for T in 1 2 4 8 16 32 64; do
    CMD="python tools/run_once.py --workload cfg2 --block $T --mode $mode --reps 1"
    $CMD > /dev/null
    ncu --metrics $M --clock-control none -k regex:"ffma|tc_layer" --csv --log-file $OUT/${mode}_T$T.csv $CMD > /dev/null
  done
done
echo done
