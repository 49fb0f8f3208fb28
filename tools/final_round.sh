#!/bin/bash
# End-of-session evidence pass on one GPU: GPU tests, smoke, default bench line
# (with the CPU baseline), reference arm, config matrix, c4 streams, formats,
# then the c2 launch list and one full ncu capture.  Everything into gpurun_out/.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu_final.log 2>&1; tail -1 gpurun_out/pytest_gpu_final.log
python __graft_entry__.py > gpurun_out/smoke_final.log 2>&1; tail -2 gpurun_out/smoke_final.log
python bench.py > gpurun_out/bench_default_final.json 2> gpurun_out/bench_default_final.err; tail -1 gpurun_out/bench_default_final.json | cut -c1-160
python bench.py --impl reference > gpurun_out/bench_reference_final.json 2> gpurun_out/bench_reference_final.err; tail -1 gpurun_out/bench_reference_final.json | cut -c1-160
bash tools/bench_matrix.sh; wc -l gpurun_out/matrix.jsonl
python bench.py --preset hq --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_c2_hq_final.json
python tools/bench_streams.py --streams 32 --frames 32 2>/dev/null | tail -1 > gpurun_out/bench_c4_streams_final.jsonl
python tools/bench_formats.py 2>/dev/null > gpurun_out/bench_formats_final.jsonl
bash tools/profile_c2.sh
