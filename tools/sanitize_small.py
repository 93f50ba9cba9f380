"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

Builds a 30k x 256 index (device input), answers 24 queries (walks + noisy copies) with the
leaf scan and the flat scan, runs an overflow-round case, and checks the ids against the oracle.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
from oracle import clib  # noqa: E402
from paper_2009_01614_b200 import isax  # noqa: E402

wl = datagen.Workload("san", 30_000, 256, 24, "walk", 21, 22, 12, 12, 0.1)
x = datagen.series(wl, 0, wl.N)
q, _ = datagen.queries(wl)
qy, _, _, _, _ = clib.summarise(q.cpu().numpy(), want_paa=False)
sc = clib.NN1Scan(qy)
sc.feed(0, x.cpu().numpy())
ids_or, _, _ = sc.result()
for opts in ({}, {"flags": 1}, {"cand_cap": 64}):
    with isax.Index.build(x, **opts) as ix:
        ids, dist = ix.nn1(q)
        torch.cuda.synchronize()
        assert np.array_equal(ids.cpu().numpy(), ids_or), opts
print("sanitize run ok")
