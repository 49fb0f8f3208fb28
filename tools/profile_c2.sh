#!/bin/bash
# Profiling pass of the default bench workload (c2 log) on one GPU:
#  1. the plain bench line (no profiler)          -> gpurun_out/prof_plain.json
#  2. the launch list (gpu__time_duration only)   -> gpurun_out/launches.csv
#  3. one --set full capture of every kernel of one push (the second; a dense
#     c2 push = 33 launches: init_ref, 3 pyramid, 4 x 3 LK levels, segments,
#     4 x (chain, offsets, segbase, emit) sub-batches)
#                                                 -> gpurun_out/prof_all.ncu-rep
# Summarise here with: python tools/ncu_summary.py gpurun_out/prof_all.ncu-rep profiles/r01
set -e
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-}"
timeout 600 python bench.py $ARGS > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err
tail -1 gpurun_out/prof_plain.json | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py $ARGS > gpurun_out/launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-pyramid|quad_level0|init_ref|dense_lk|segments|chain|offsets|segbase|emit}" \
  --launch-skip ${SKIP:-33} -c ${COUNT:-33} -f -o gpurun_out/prof_all \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/prof_all.log 2>&1
echo profile done
