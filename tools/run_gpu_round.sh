#!/bin/bash
# One GPU session: tests, smoke, bench lines. Usage: bash tools/run_gpu_round.sh <tag> [configs...]
tag=${1:-r}; shift
cfgs=${@:-"2 3"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_gpu.txt
timeout 420 python -m pytest tests -q -m gpu -x > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 150 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
for c in $cfgs; do
  timeout 240 python bench.py --config $c --steps 20 --warmup 3 --stats-out gpurun_out/${tag}_stats_cfg$c.json > gpurun_out/${tag}_bench_cfg$c.json 2> gpurun_out/${tag}_bench_cfg$c.err; echo "bench cfg$c rc=$?" >> gpurun_out/${tag}_bench_cfg$c.err
done
tail -3 gpurun_out/${tag}_pytest.log; tail -2 gpurun_out/${tag}_smoke.log; for c in $cfgs; do cat gpurun_out/${tag}_bench_cfg$c.json; tail -3 gpurun_out/${tag}_bench_cfg$c.err; done
