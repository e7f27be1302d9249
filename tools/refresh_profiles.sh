#!/bin/bash
# One gpurun call that regenerates the judged evidence under gpurun_out/:
#   bench_c2.json (driver-default bench incl. CPU baseline), bench_ref.json
#   (reference arm), bench_c3.json (Transformer-XL base), launches_c2.csv
#   (ncu launch list of bench steps), head_full.ncu-rep (ncu --set full of the
#   four head GEMMs).  Each ncu pass runs only after its command exited 0.
set -u
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --config c3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
      --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
REPS=1 python tools/prof_head.py > /dev/null 2>&1 && \
  REPS=1 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -c 4 \
      -o gpurun_out/head_full python tools/prof_head.py > gpurun_out/ncu_head.log 2>&1
tail -c 400 gpurun_out/bench_c2.json; echo; tail -c 300 gpurun_out/bench_ref.json; echo; tail -c 300 gpurun_out/bench_c3.json
