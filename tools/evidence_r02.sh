#!/bin/bash
# Round-2 evidence pass on one GPU.  Small outputs only into gpurun_out/ev_*
# (gpurun copies back <= 64 MiB): the ncu reports stay in /tmp on the box and
# are summarised there (tools/ncu_summary.py, tools/ncu_source_hot.py).
#  1. the default bench line (c5 log) and the reference arm beside it
#  2. every BASELINE config (with the CPU baseline), stacked c1 x64, c4's 32
#     streams; reference-arm lines for c1 - c4            (PART=bench)
#  3. the launch list of the default command, ncu --set full of one c5 push's
#     kernels and of the stacked c1 push                     (PART=ncu)
set -x
mkdir -p gpurun_out
B="python bench.py"
if [ "${PART:-bench}" = bench ]; then
timeout 900 $B > gpurun_out/ev_default.json 2> gpurun_out/ev_default.err
timeout 900 $B --impl reference > gpurun_out/ev_reference_c5.json 2> gpurun_out/ev_reference_c5.err
: > gpurun_out/ev_matrix.jsonl
for a in "--config c1 --mode log" "--config c1 --mode linear" "--config c1 --mode log --streams 64" \
         "--config c1 --mode linear --streams 64" "--config c2 --mode log" "--config c2 --mode linear" \
         "--config c3 --mode log" "--config c3 --mode linear" "--config c4 --mode log" "--config c5 --mode linear" \
         "--config c2 --mode log --preset hq"; do
  timeout 1200 $B $a --steps 3 --warmup 3 2>> gpurun_out/ev_matrix.err | tail -1 >> gpurun_out/ev_matrix.jsonl
done
: > gpurun_out/ev_reference.jsonl
for a in "--config c1 --mode log" "--config c1 --mode log --streams 64" "--config c2 --mode log" "--config c3 --mode log" \
         "--config c4 --mode log"; do
  timeout 900 $B --impl reference $a --steps 3 --warmup 1 2>> gpurun_out/ev_reference.err | tail -1 >> gpurun_out/ev_reference.jsonl
done
fi
if [ "${PART:-bench}" = ncu ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_c5.csv \
  $B --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/ev_launches_c5.log 2>&1
python tools/launch_summary.py gpurun_out/ev_launches_c5.csv > gpurun_out/ev_launches_c5.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"chain_dense|lerp_quad|dense_lk_warp|emit|quad_level0|pyramid|offsets|segbase|segments|init_ref" \
  --launch-skip 0 -c 60 -f -o /tmp/ev_full_c5 python tools/push_once.py c5 log 7 1 > gpurun_out/ev_full_c5.log 2>&1
# the second push (7 pairs) is the one summarised: drop the first push's launches by taking the last ones
python tools/ncu_summary.py /tmp/ev_full_c5.ncu-rep gpurun_out/ev_full_c5 c5:log:7 > gpurun_out/ev_full_c5.txt 2>&1
for k in chain_dense dense_lk_warp emit_single lerp_quad; do
  python tools/ncu_source_hot.py /tmp/ev_full_c5.ncu-rep $k 25 > gpurun_out/ev_hot_c5_$k.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"chain_diff|emit" --launch-skip 6 -c 4 \
  -f -o /tmp/ev_full_c1x64 $B --config c1 --mode log --streams 64 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline \
  --no-parity > gpurun_out/ev_full_c1x64.log 2>&1
python tools/ncu_summary.py /tmp/ev_full_c1x64.ncu-rep gpurun_out/ev_full_c1x64 c1x64:log:63 > gpurun_out/ev_full_c1x64.txt 2>&1
python tools/ncu_source_hot.py /tmp/ev_full_c1x64.ncu-rep chain_diff 25 > gpurun_out/ev_hot_c1x64.txt 2>&1
# the opt-in tile-staged chain on the same push
EVSIM_CHAIN_QUAD=tile EVSIM_TILE_BLOCKS=4 timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"chain_dense_tile" --launch-skip 1 -c 1 -f -o /tmp/ev_tile_c5 python tools/push_once.py c5 log 7 1 \
  > gpurun_out/ev_tile_c5.log 2>&1
python tools/ncu_kernel_metrics.py /tmp/ev_tile_c5.ncu-rep > gpurun_out/ev_tile_c5.txt 2>&1
python tools/ncu_kernel_metrics.py /tmp/ev_full_c1x64.ncu-rep chain_diff > gpurun_out/ev_c1x64_diff_chain.txt 2>&1
python tools/ncu_kernel_metrics.py /tmp/ev_full_c5.ncu-rep > gpurun_out/ev_full_c5_metrics.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"chain_dense" --launch-skip 1 -c 1 \
  -f -o gpurun_out/ev_chain_c5 python tools/push_once.py c5 log 7 1 > gpurun_out/ev_chain_c5.log 2>&1
fi
du -sh gpurun_out
echo evidence done
