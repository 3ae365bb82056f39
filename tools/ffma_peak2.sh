#!/bin/bash
# FMA peak cross-check with SM clocks sampled while it runs.
nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active,power.draw --format=csv,noheader -lms 200 > gpurun_out/ffma_peak2_clocks.csv &
S=$!
./tools/ffma_peak2 | tee gpurun_out/ffma_peak2.txt
kill $S
sort gpurun_out/ffma_peak2_clocks.csv | uniq -c | sort -rn | head -8
