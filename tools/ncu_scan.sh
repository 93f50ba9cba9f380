#!/bin/bash
# One ncu --set full capture of the leaf scan (third launch: a full scan, first band off) per config.
# Usage: bash tools/ncu_scan.sh <tag> "<configs>"
tag=$1; cfgs=$2
mkdir -p gpurun_out
for c in $cfgs; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'itemscan|leafscan' -s 2 -c 1 -f -o gpurun_out/${tag}_leafscan$c \
    python tools/sweep_env.py --config $c --steps 2 --opt first_band=-1 > gpurun_out/${tag}_ncu$c.log 2>&1
  echo "ncu cfg$c rc=$?"
done
