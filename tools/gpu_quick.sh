# quick GPU check: a subset of the GPU tests, then a few bench lines (value, e2e, stage split)
set -e
python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "${K:-dense or random or parity or stream or band or flow or lk}" 2>&1 | tail -3
for cm in ${CFGS:-c2:log c2:linear c3:log}; do
  c=${cm%%:*}; m=${cm##*:}
  python bench.py --config $c --mode $m --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} 2>/dev/null | tail -1 \
    | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], d["value"], d["e2e"]["value"], d["roofline"].get("stage_us_per_frame"))' "$c $m"
done
