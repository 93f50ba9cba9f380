#!/bin/bash
# Round 2c evidence in one GPU call: bench lines, launch lists, and ncu --set full captures of the
# scan kernels, the refine passes, the window kernel and the summarise kernel.
set -x
mkdir -p gpurun_out
T=r02c
for c in 3 2 4 5 1; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/${T}_bench_cfg$c.json 2> gpurun_out/${T}_bench_cfg$c.err
done
for c in 3 5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/${T}_launches_cfg$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_l$c.log 2>&1
done
# third scan launch of a sweep_env run = a full scan with the first band off
for c in 3 2 5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:itemscan -s 2 -c 1 -f -o gpurun_out/${T}_itemscan$c \
    python tools/sweep_env.py --config $c --steps 2 --opt first_band=-1 > gpurun_out/${T}_ncu_i$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nodescan -s 2 -c 1 -f -o gpurun_out/${T}_nodescan3 \
  python tools/sweep_env.py --config 3 --steps 2 --opt first_band=-1 > gpurun_out/${T}_ncu_n3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'refine_q|filter' -s 3 -c 3 -f -o gpurun_out/${T}_refine3 \
  python tools/sweep_env.py --config 3 --steps 2 --opt first_band=-1 > gpurun_out/${T}_ncu_r3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:window_kernel -s 1 -c 1 -f -o gpurun_out/${T}_window3 \
  python tools/sweep_env.py --config 3 --steps 2 --opt first_band=-1 > gpurun_out/${T}_ncu_w3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:candcheck -s 1 -c 1 -f -o gpurun_out/${T}_candcheck3 \
  python tools/sweep_env.py --config 3 --steps 2 --opt first_band=-1 > gpurun_out/${T}_ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'summarise_tma|superkd' -c 2 -f -o gpurun_out/${T}_build2 \
  python tools/time_build.py --config 2 --reps 1 > gpurun_out/${T}_ncu_b2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_build_launches_cfg2.csv \
  python tools/time_build.py --config 2 --reps 1 > gpurun_out/${T}_ncu_bl2.log 2>&1
python tools/time_build.py --config 2 --reps 3 > gpurun_out/${T}_build_cfg2.txt 2>&1
python tools/time_build.py --config 3 --reps 1 > gpurun_out/${T}_build_cfg3.txt 2>&1
ls -la gpurun_out | tail -40
