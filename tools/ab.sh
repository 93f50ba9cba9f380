#!/bin/bash
# A/B of library variants: bash tools/ab.sh <tag> "<configs>" <variant> [<variant> ...]
# variant "main" = the in-tree libisax.so, "name" = variants/<name>/libisax.so;
# append ":k=v,k=v" for index options (e.g. main:flags=2)
tag=$1; cfgs=$2; shift 2
mkdir -p gpurun_out
for c in $cfgs; do
  for vv in "$@"; do
    v=${vv%%:*}; o=""; [ "$vv" != "$v" ] && o=${vv#*:}
    if [ "$v" = main ]; then lib=""; else lib=variants/$v/libisax.so; fi
    args=""; for kv in ${o//,/ }; do args="$args --opt $kv"; done
    name=$(echo "$vv" | tr ':,=' '___')
    ISAX_LIB=$lib timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline $args > gpurun_out/${tag}_${name}_cfg$c.json 2> gpurun_out/${tag}_${name}_cfg$c.err
    python -c "
import json,sys
d=json.load(open('gpurun_out/${tag}_${name}_cfg$c.json'))
print('cfg$c', '$vv'.ljust(16), round(d['value']), 'q/s', d['ms_per_step'], 'ms', {k: v for k, v in d['kernels']['ms_first_batch'].items()}, 'e2e', round(d['e2e']['value']), d['stats'])" || tail -3 gpurun_out/${tag}_${name}_cfg$c.err
  done
done
