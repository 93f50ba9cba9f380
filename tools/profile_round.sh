set -x
bash tools/run_gpu_round.sh r02q 3 2 4 5 1 > gpurun_out/r02q_round.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/r02q3_launches.csv python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02q3_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/r02q5_launches.csv python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02q5_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'refine_q|filter' -s 3 -c 3 -o gpurun_out/r02q_refine3 python tools/sweep_env.py --config 3 --steps 2 --opt first_band=-1 > gpurun_out/r02q_ref3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'refine_q|filter' -s 3 -c 3 -o gpurun_out/r02q_refine4 python tools/sweep_env.py --config 4 --steps 2 --opt first_band=-1 > gpurun_out/r02q_ref4.log 2>&1
ls gpurun_out
