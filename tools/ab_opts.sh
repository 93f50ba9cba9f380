#!/bin/bash
# A/B of index options on the in-tree library: bash tools/ab_opts.sh "<configs>" "<k=v,k=v>" ["<k=v>" ...]
# ("-" = library defaults). Prints q/s, stage ms and counters of bench.py runs (30 steps).
cfgs=$1; shift
mkdir -p gpurun_out
for c in $cfgs; do
  for o in "$@"; do
    args=""; [ "$o" != "-" ] && for kv in ${o//,/ }; do args="$args --opt $kv"; done
    timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline $args > gpurun_out/abo.json 2> gpurun_out/abo.err
    python -c "
import json
d=json.load(open('gpurun_out/abo.json'))
print('cfg$c', '$o'.ljust(22), round(d['value']), 'q/s', d['ms_per_step'], 'ms', d['kernels']['ms_first_batch'], 'cand', round(d['stats']['candidates_per_query']), 'rounds', d['stats']['rounds_max'])" || tail -3 gpurun_out/abo.err
  done
done
