#!/bin/bash
# Where the tcgen05 layer kernel's time goes: the same forward with parts of
# the pipeline switched off (RNNB_DEBUG bits, timing only -- results wrong):
# 32 = epilogue only hands accumulators back, 64 = no MMAs, 128 = no TMA loads.
for dbg in 0 32 64 96 128 160 192; do
  echo "== RNNB_DEBUG=$dbg"
  RNNB_DEBUG=$dbg python tools/time_layer.py --workload ${1:-cfg2} --mode ${2:-bf16} --blocks ${3:-16,32,64} --reps 20
done
