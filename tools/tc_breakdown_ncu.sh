#!/bin/bash
# Device time of the tcgen05 layer kernel alone (ncu gpu__time_duration, one
# launch per variant; the host-side launch floor of a python loop hides
# sub-30-us kernels from CUDA-event timing) with parts of the pipeline off:
# RNNB_DEBUG 16 no look-back, 32 no epilogue, 64 no MMAs, 128 no loads,
# 512 no scan/stores, 1024 no activations (timing only: results wrong).
W=${1:-cfg2}; M=${2:-bf16}; BL=${3:-16 32 64}
for T in $BL; do
  for dbg in 0 16 32 64 96 128 160 192 208 704 1216 1744 512 1024 528; do
    RNNB_DEBUG=$dbg python tools/run_once.py --workload $W --mode $M --block $T --reps 2 > /dev/null || exit 1
    RNNB_DEBUG=$dbg ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_layer -s 1 -c 1 --csv \
      python tools/run_once.py --workload $W --mode $M --block $T --reps 2 2>/dev/null | \
      awk -v T=$T -v d=$dbg -F'","' '/gpu__time_duration/ {gsub(/"/,"",$NF); print "T_b=" T " dbg=" d " us=" $NF/1000}'
  done
done
