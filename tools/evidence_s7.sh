#!/bin/bash
# Evidence pass of the round's last session (the tap-relative lerp quads): the
# full GPU tests, the default bench line, its ncu launch list, and ncu --set
# full of one c5 push (traffic / instruction counts read by bench.py).
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/s8_pytest.log 2>&1; tail -2 gpurun_out/s8_pytest.log
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"chain_dense|lerp_quad|dense_lk_warp|emit|quad_level0|pyramid|offsets|segbase|segments|init_ref" \
  --launch-skip 0 -c 60 -f -o /tmp/ev_full_c5 python tools/push_once.py c5 log 7 1 > gpurun_out/s8_full_c5.log 2>&1
python tools/ncu_summary.py /tmp/ev_full_c5.ncu-rep gpurun_out/s8_full_c5 c5:log:7 > gpurun_out/s8_full_c5.txt 2>&1
python tools/ncu_source_hot.py /tmp/ev_full_c5.ncu-rep chain_dense 25 > gpurun_out/s8_hot_c5_chain_dense.txt 2>&1
python tools/ncu_kernel_metrics.py /tmp/ev_full_c5.ncu-rep > gpurun_out/s8_full_c5_metrics.txt 2>&1
cp gpurun_out/s8_full_c5/traffic_c5_log.json profiles/r02/traffic_c5_log.json
timeout 900 python bench.py > gpurun_out/s8_default.json 2> gpurun_out/s8_default.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s8_launches_c5.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/s8_launches_c5.log 2>&1
python tools/launch_summary.py gpurun_out/s8_launches_c5.csv > gpurun_out/s8_launches_c5.txt 2>&1
tail -c 400 gpurun_out/s8_default.json
echo evidence done
