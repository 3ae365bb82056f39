#!/bin/bash
# Round-2 evidence on one GPU: the ncu launch list of the bench command and
# one full ncu capture of each headline tcgen05 kernel (fp32-accurate 3xTF32
# at cfg2 T_b=32 = the bench headline; bf16 at T_b=64), plus the per-T_b
# counter sweep.  Each command first runs plainly (must exit 0).  The launch
# list leaves the host-buffer (e2e) and drop-in legs out (--no-e2e
# --no-dropin): ncu serialises kernels, so the streaming host path (a
# conversion kernel feeding a running layer kernel) would only show its 2 s
# input time-out before falling back to the chunked path.
set -x
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-sweep --extra-modes '' --no-cpu-baseline --no-configs --no-partitioned --no-e2e --no-dropin > gpurun_out/b_small.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2.csv \
    python bench.py --steps 2 --warmup 3 --no-sweep --extra-modes '' --no-cpu-baseline --no-configs --no-partitioned --no-e2e --no-dropin > gpurun_out/ncu_l.log 2>&1
python tools/run_once.py --workload cfg2 --mode f32 --block 32 --reps 1 > /dev/null && \
  ncu --set full --import-source on --clock-control none -k regex:tc_layer -c 1 -f -o gpurun_out/prof_r2_tc_f32x3_cfg2_T32 \
    python tools/run_once.py --workload cfg2 --mode f32 --block 32 --reps 1 > gpurun_out/ncu_f1.log 2>&1
python tools/run_once.py --workload cfg2 --mode bf16 --block 64 --reps 1 > /dev/null && \
  ncu --set full --import-source on --clock-control none -k regex:tc_layer -c 1 -f -o gpurun_out/prof_r2_tc_bf16_cfg2_T64 \
    python tools/run_once.py --workload cfg2 --mode bf16 --block 64 --reps 1 > gpurun_out/ncu_f2.log 2>&1
bash tools/ncu_sweep.sh gpurun_out/ncu_sweep_r2 > gpurun_out/ncu_sweep_r2.log 2>&1
echo done
