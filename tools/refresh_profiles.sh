#!/bin/bash
# One gpurun call that regenerates the judged evidence under gpurun_out/:
#   bench_c2.json (driver-default bench incl. CPU baseline), bench_ref.json
#   (reference arm), bench_c3.json (Transformer-XL base), launches_c2.csv /
#   launches_c3.csv (ncu launch lists of bench steps), head_full.ncu-rep (ncu
#   --set full of the four head GEMMs), xl_attn_full.ncu-rep (the fused XL
#   attention kernels).  Each ncu pass runs only after its command exited 0.
set -u
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --config c3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --steps 2 --warmup 1 --no-cpu --no-compare-k1 > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
      --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-compare-k1 > gpurun_out/ncu_launch.log 2>&1
python bench.py --config c3 --steps 2 --warmup 1 --no-cpu --no-compare-k1 > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
      --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 1 --no-cpu --no-compare-k1 > gpurun_out/ncu_launch_c3.log 2>&1
REPS=1 python tools/prof_head.py > /dev/null 2>&1 && \
  REPS=1 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -c 4 \
      -o gpurun_out/head_full python tools/prof_head.py > gpurun_out/ncu_head.log 2>&1
REPS=1 python tools/prof_xl_attn.py > gpurun_out/xl_attn_timing.txt 2>&1 && \
  REPS=1 ncu --set full --import-source on --clock-control none -k regex:xl_attn -c 2 \
      -o gpurun_out/xl_attn_full python tools/prof_xl_attn.py > gpurun_out/ncu_xl_attn.log 2>&1
python tools/launches.py gpurun_out/launches_c2.csv > gpurun_out/launches_c2_summary.txt
python tools/launches.py gpurun_out/launches_c3.csv > gpurun_out/launches_c3_summary.txt
tail -c 400 gpurun_out/bench_c2.json; echo; tail -c 300 gpurun_out/bench_ref.json; echo; tail -c 300 gpurun_out/bench_c3.json
cat gpurun_out/xl_attn_timing.txt
