#!/bin/bash
# ncu evidence for one bench command. Usage: bash tools/profile_gpu.sh <tag> <config> [kernel-regex]
tag=${1:-r}; cfg=${2:-3}; kre=${3:-lbscan}
mkdir -p gpurun_out
CMD="python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/${tag}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/${tag}_launches.csv $CMD > gpurun_out/${tag}_ncu_launches.log 2>&1
echo "launches rc=$?"
$CMD > gpurun_out/${tag}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$kre -s 0 -c 1 -o gpurun_out/${tag}_prof $CMD > gpurun_out/${tag}_ncu_full.log 2>&1
echo "full rc=$?"
tail -3 gpurun_out/${tag}_ncu_full.log
