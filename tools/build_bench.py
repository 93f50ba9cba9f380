"""Time the build stages of one BASELINE config on the GPU (device-resident input when it fits).

python tools/build_bench.py --config 2
Prints one JSON line: build seconds, summarise/sort/permute ms from a CUDA-event trace.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2009_01614_b200 import isax  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
wl = datagen.WORKLOADS[a.config]
x = datagen.series(wl, 0, wl.N)
torch.cuda.synchronize()
times = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ix = isax.Index.build(x)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
    ix.close()
print(json.dumps({"config": wl.name, "build_ms": times, "input_GB": wl.N * wl.n * 4 / 1e9,
                  "GBps_best": wl.N * wl.n * 4 / 1e9 / (min(times) / 1e3)}))
