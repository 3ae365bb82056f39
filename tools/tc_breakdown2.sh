#!/bin/bash
# Epilogue composition of the tcgen05 layer kernel with the MMAs and loads off
# (RNNB_DEBUG 192): + 16 no look-back, + 512 no scan/stores, + 1024 no activations.
for dbg in 192 208 704 1216 720 1232 1728 1744 0 16; do
  echo "== RNNB_DEBUG=$dbg"
  RNNB_DEBUG=$dbg python tools/time_layer.py --workload ${1:-cfg2} --mode ${2:-bf16} --blocks ${3:-16,32,64} --reps 20
done
