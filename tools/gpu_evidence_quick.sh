#!/bin/bash
# One GPU session of round evidence at HEAD: bench (ours + reference arm), the
# ncu launch list of the bench command, one full ncu capture of the headline
# kernel, and every BASELINE config (incl. the emulated P2P partitions).
# Outputs under gpurun_out/ (copy what is judged to profiles/).
set -x
python bench.py > gpurun_out/bench_r1g.json 2> gpurun_out/bench_r1g.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_g.json 2>&1
python bench.py --steps 2 --warmup 3 --no-sweep --extra-modes '' --no-cpu-baseline > gpurun_out/b_small.json 2>&1 && \
  RNNB_HOST_STREAM=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_g.csv python bench.py --steps 2 --warmup 3 --no-sweep --extra-modes '' --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
python tools/run_once.py --reps 1 > /dev/null && ncu --set full --import-source on --clock-control none -k regex:ffma_ws -c 1 -f -o gpurun_out/prof_r1g_ffma_cfg2_T32 python tools/run_once.py --reps 1 > gpurun_out/ncu_f.log 2>&1
python tools/bench_configs.py --p2p --out gpurun_out/configs_g.json > gpurun_out/configs_g.log 2>&1
echo done
