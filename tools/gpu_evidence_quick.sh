set -x
python bench.py > gpurun_out/bench_r1f.json 2> gpurun_out/bench_r1f.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_f.json 2>&1
python bench.py --steps 2 --warmup 3 --no-sweep --extra-modes '' --no-cpu-baseline > gpurun_out/b_small.json 2>&1 && \
  RNNB_HOST_STREAM=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_f.csv python bench.py --steps 2 --warmup 3 --no-sweep --extra-modes '' --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
python tools/run_once.py --reps 1 > /dev/null && ncu --set full --import-source on --clock-control none -k regex:ffma_ws -c 1 -f -o gpurun_out/prof_r1f_ffma_cfg2_T32 python tools/run_once.py --reps 1 > gpurun_out/ncu_f.log 2>&1
echo done
