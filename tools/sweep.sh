#!/bin/bash
# Option sweep at one config: bash tools/sweep.sh <tag> <config> "<opts1>" "<opts2>" ...
# each opts string is space-separated key=value pairs passed as --opt to bench.py
tag=$1; cfg=$2; shift 2
mkdir -p gpurun_out
i=0
for o in "$@"; do
  args=""; for kv in $o; do args="$args --opt $kv"; done
  timeout 240 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline $args > gpurun_out/${tag}_$i.json 2> gpurun_out/${tag}_$i.err
  echo "$i [$o] rc=$?"; i=$((i+1))
done
