#!/bin/bash
# Run bench.py over the BASELINE configs in both contrast modes; one JSON line
# per run in gpurun_out/matrix.jsonl (used for DESIGN.md §6's table).
out=gpurun_out/matrix.jsonl
mkdir -p gpurun_out
: > $out
for cm in "c1 log" "c1 linear" "c2 log" "c2 linear" "c3 log" "c3 linear" "c5 log" "c5 linear"; do
  set -- $cm
  timeout 900 python bench.py --config $1 --mode $2 --steps 3 --warmup 3 --no-cpu-baseline \
    2> gpurun_out/matrix_$1_$2.err | tail -1 >> $out
done
