"""Helpers for the GPU parity tests: generator -> device build, oracle on the same bytes."""
from __future__ import annotations

import numpy as np

import datagen
from oracle import clib, ref


def small_workload(N, n, kind="walk", seed=11, Q=8, q_seed=12, q_noisy=0, sigma=0.1):
    return datagen.Workload(f"test_{kind}_{N}x{n}", N, n, Q, kind, seed, q_seed, Q - q_noisy, q_noisy, sigma)


def device_data(wl):
    return datagen.series(wl, 0, wl.N)


def oracle_nn1(x_host: np.ndarray, q_host: np.ndarray, chunk: int = 1 << 20, K: int = 32):
    """Exact 1-NN by the C oracle (brute force over raw rows; z-norm inside), same bytes as the GPU."""
    qy, _, _, _, _ = clib.summarise(q_host, want_paa=False)
    sc = clib.NN1Scan(qy, K=K)
    for s in range(0, x_host.shape[0], chunk):
        sc.feed(s, x_host[s : s + chunk])
    return sc.result()


def oracle_nn1_streamed(wl, q_host: np.ndarray, chunk: int = 1 << 21, K: int = 32):
    """Exact 1-NN over a workload too big for host RAM: regenerate chunks on the device, copy each to host."""
    import torch

    qy, _, _, _, _ = clib.summarise(q_host, want_paa=False)
    sc = clib.NN1Scan(qy, K=K)
    buf = torch.empty((chunk, wl.n), dtype=torch.float32, device="cuda")
    host = torch.empty((chunk, wl.n), dtype=torch.float32, pin_memory=True)
    for s in range(0, wl.N, chunk):
        c = min(chunk, wl.N - s)
        datagen.series(wl, s, c, out=buf[:c])
        host[:c].copy_(buf[:c])
        sc.feed(s, host[:c].numpy())
    return sc.result()


def assert_nn_parity(ids_gpu, dist_gpu, ids_or, dist_or, rel=1e-5):
    ids_gpu = np.asarray(ids_gpu)
    dist_gpu = np.asarray(dist_gpu, dtype=np.float64)
    bad = np.nonzero(ids_gpu != ids_or)[0]
    assert bad.size == 0, f"id mismatch at queries {bad[:10]}: gpu {ids_gpu[bad[:10]]} oracle {ids_or[bad[:10]]}"
    err = np.abs(dist_gpu - dist_or) / np.maximum(np.abs(dist_or), 1e-3)
    assert np.all(err <= rel), f"dist rel err max {err.max()} at {np.argmax(err)}"
