"""The N > 1 bench path on CPU: 2 ranks over gloo (replicas only).

Each rank answers its own query batch; the oracle stands in for the device on CPU. The test
checks three things:
* the per-rank workloads differ only in the query seed;
* the timing reduction takes the max over ranks;
* the aggregate counts every rank's queries over the slowest rank's time.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import datagen
    from datagen import host
    from oracle import ref
    from paper_2009_01614_b200 import dist as pdist

    wl = pdist.rank_workload(datagen.WORKLOADS[1], rank)
    # a tiny replica of the collection (same on every rank) and this rank's queries
    x = host.walks(2000, 64, 1)
    q = host.walks(4, 64, wl.q_seed)
    ids, _ = ref.nn1_index_search(x, q, 16, 256)
    ms = 10.0 + 5.0 * rank  # stand-in device time of this rank
    mx = pdist.max_over_ranks(ms)
    qps = pdist.aggregate_qps(len(q), 3, world, mx)
    out[rank] = (wl.q_seed, mx, qps, ids.tolist())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replicas_over_gloo():
    world, port = 2, _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    (s0, mx0, q0, ids0), (s1, mx1, q1, ids1) = res[0], res[1]
    assert s0 != s1  # each rank answers its own queries
    assert mx0 == mx1 == 15.0  # max over ranks
    assert q0 == q1 == pytest.approx(4 * 3 * 2 / 0.015)
    # each rank's answers are exact (index search == brute force, the oracle's own pin)
    from datagen import host
    from oracle import ref

    x = host.walks(2000, 64, 1)
    for seed, ids in ((s0, ids0), (s1, ids1)):
        q = host.walks(4, 64, seed)
        Y, _, _ = ref.znorm(x)
        qy, _, _ = ref.znorm(q)
        bf, _, _ = ref.nn1_bruteforce(Y, qy)
        np.testing.assert_array_equal(bf, ids)
