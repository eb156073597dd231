#!/bin/bash
# Every bench line kept under profiles/ (one B200): bash scripts/bench_all.sh OUTDIR TAG
# -> OUTDIR/TAG_bench_<name>.json (the JSON line; stderr in .err)
OUT=${1:-gpurun_out}; TAG=${2:-rX}
cd "$(dirname "$0")/.."
run() { name=$1; shift; timeout 900 python bench.py "$@" > "$OUT/${TAG}_bench_$name.json" 2> "$OUT/${TAG}_bench_$name.err"; }
run c2 --steps 10 --warmup 3
run c2_fp32 --steps 10 --warmup 3 --precision fp32 --no-variants
run c2_p350k --steps 5 --warmup 3 --model p350k --no-variants
run c2_pool_meta --steps 10 --warmup 3 --model pool-meta --no-variants
run c3 --config C3 --steps 10 --warmup 3
run c3_p12 --config C3 --model p12 --steps 5 --warmup 3
run c3_volume --config C3 --model 3d --steps 10 --warmup 3
run c3_pool_meta --config C3 --model pool-meta --steps 10 --warmup 3
run c4 --config C4 --steps 10 --warmup 3
run c5 --config C5 --steps 5 --warmup 3
