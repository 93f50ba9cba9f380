#!/bin/bash
# ncu evidence for one bench command: the launch list of the whole run and one --set full
# capture per kernel regex. Usage: bash tools/profile_gpu.sh <tag> <config> <regex> [<regex> ...]
tag=${1:-r}; cfg=${2:-3}; shift 2
mkdir -p gpurun_out
CMD="python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/${tag}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/${tag}_launches.csv $CMD > gpurun_out/${tag}_ncu_launches.log 2>&1
echo "launches rc=$?"
for kre in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:$kre -s 0 -c 1 -o gpurun_out/${tag}_${kre}_prof $CMD > gpurun_out/${tag}_${kre}_ncu_full.log 2>&1
  echo "full $kre rc=$?"
done
