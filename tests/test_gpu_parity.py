"""GPU parity: the CUDA path (through the C-ABI) against the oracle on the same seeded bytes.

Bars:
* iSAX words and the stored z-normalised rows: bit-exact; the permutation: the layout properties
  of tests/layout_props.py (C5 blocks, kd splits), not a restatement of the kernels' rule.
* query PAA and word: bit-exact; LB^2: within the fp32 summation bound of the fp64 oracle.
* NN ids: exact (ties to the lowest id); distances within 1e-5 relative (north_star).
Sizes span many tiles and a ragged tail; edge cases cover N = 1, N < window, duplicates,
constant series, exact-copy queries, overflow rounds and batch splitting.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import datagen  # noqa: E402
from oracle import clib, ref  # noqa: E402
from paper_2009_01614_b200 import isax  # noqa: E402
from tests import layout_props  # noqa: E402
from tests.gpu_util import assert_nn_parity, oracle_nn1, small_workload  # noqa: E402


def _build(x, **opts):
    return isax.Index.build(x, **opts)


@pytest.mark.parametrize("N,n,kind", [(100_000, 256, "walk"), (12_345, 128, "walk"), (4_099, 64, "sines"), (1, 256, "walk"),
                                      (1_024, 256, "walk"), (3_072, 128, "sines"), (1_025, 256, "walk"),
                                      (2_500, 1024, "walk"), (3_333, 512, "sines")])
def test_summaries_perm_and_rows_bit_exact(N, n, kind):
    wl = small_workload(N, n, kind)
    x = datagen.series(wl, 0, N)
    xh = x.cpu().numpy()
    with _build(x) as ix:
        ex = ix.export(0, N, sax=True, perm=True, stored=True)
    y, mu, sd, m, word = clib.summarise(xh)
    np.testing.assert_array_equal(ex["sax"], word)  # C4 words, by id
    perm = ex["perm"].astype(np.int64)
    # the layout's properties (tests/layout_props.py): a bijection, super-nodes = the C5 blocks,
    # kd splits on each node's widest segment, stable (R6, R6b)
    layout_props.check_layout(perm, word)
    np.testing.assert_array_equal(ex["stored"], y[perm])  # C1 rows, in the sorted order


@pytest.mark.parametrize("N,n", [(100_000, 256), (9_999, 128), (3_072, 256), (1_500, 128)])
def test_query_summary_lb_and_window(N, n):
    wl = small_workload(N, n, Q=16)
    x = datagen.series(wl, 0, N)
    q, _ = datagen.queries(wl)
    xh, qh = x.cpu().numpy(), q.cpu().numpy()
    with _build(x) as ix:
        ex = ix.export(0, N, sax=True, perm=True)
        dbg = ix.query_debug(qh, 0, N)
    _, _, _, qm, qw = clib.summarise(qh)
    np.testing.assert_array_equal(dbg["q_paa"], qm)
    np.testing.assert_array_equal(dbg["q_sax"], qw)
    words_sorted = ex["sax"][ex["perm"]]
    for i in range(len(qh)):
        lb_or = ref.lb2(qm[i], words_sorted, n)  # C6, fp64
        lb_gpu = dbg["lb2"][i].astype(np.float64)
        # fp32 sum of 16 rounded-down terms: never above the fp64 bound beyond summation error
        assert np.all(lb_gpu <= lb_or * (1 + 2e-6) + 1e-30)
        assert np.all(lb_gpu >= lb_or * (1 - 1e-5) - 1e-6)
        layout_props.check_window(dbg["win"][i], ex["perm"], ex["sax"], qw[i], 3072)


@pytest.mark.parametrize("L", [1024, 2048, 4096])
def test_window_of_whole_super_nodes(L):
    """Main windows of 1, 2 or 4 super-nodes (R5, R6b): whole super-nodes holding the query key's
    predecessor (and, from two super-nodes on, its successor) in the C5 key order.
    window_L above 4096 is rejected (include/isax.h)."""
    N, n = 60_000, 128
    wl = small_workload(N, n, Q=16, q_noisy=8)
    x = datagen.series(wl, 0, N)
    q, _ = datagen.queries(wl)
    qh = q.cpu().numpy()
    with _build(x, window_L=L) as ix:
        ex = ix.export(0, N, sax=True, perm=True)
        dbg = ix.query_debug(qh, 0, 1)
    _, _, _, _, qw = clib.summarise(qh)
    for i in range(len(qh)):
        layout_props.check_window(dbg["win"][i], ex["perm"], ex["sax"], qw[i], L)
    with pytest.raises(isax.IsaxError):
        _build(x, window_L=4097)


@pytest.mark.parametrize("N,n,kind,q_noisy", [(100_000, 256, "walk", 0), (100_000, 256, "walk", 8),
                                              (20_000, 256, "sines", 16), (7_777, 128, "walk", 4),
                                              (5_000, 64, "sines", 4), (3_000, 1024, "walk", 4), (6_001, 512, "walk", 3)])
def test_nn1_matches_oracle(N, n, kind, q_noisy):
    wl = small_workload(N, n, kind, Q=16, q_noisy=q_noisy, sigma=0.1)
    x = datagen.series(wl, 0, N)
    q, src = datagen.queries(wl)
    xh, qh = x.cpu().numpy(), q.cpu().numpy()
    ids_or, dist_or, _ = oracle_nn1(xh, qh)
    with _build(x) as ix:
        ids, dist = ix.nn1(q)  # device path (isax_nn1_async)
        st = ix.stats()
        ids_h, dist_h = ix.nn1(qh)  # host path (isax_nn1)
    assert_nn_parity(ids.cpu().numpy(), dist.cpu().numpy(), ids_or, dist_or)
    np.testing.assert_array_equal(ids_h.numpy(), ids.cpu().numpy())
    np.testing.assert_array_equal(dist_h.numpy(), dist.cpu().numpy())
    for j in range(len(qh)):
        w0, w1 = st["window"][2 * j], st["window"][2 * j + 1]
        assert st["candidates"][j] + (w1 - w0) <= N
        # accounting: every candidate is refined to the end, abandoned, or skipped by the second
        # band's bound test (R14); window rows are counted apart
        assert st["refined"][j] + st["abandoned"][j] + st["skipped"][j] == st["candidates"][j]
        # window rows refined: the main window plus the kept probe windows (each at most probe_L
        # rows, none inside the main window, no repeats)
        lp = min(st["probe_L"], N)
        assert (w1 - w0) <= st["window_rows"][j] <= (w1 - w0) + st["probe_windows"] * lp
        assert (st["window_rows"][j] - (w1 - w0)) % lp == 0


@pytest.mark.parametrize("N,n,kind", [(200_000, 256, "walk"), (50_001, 128, "walk"), (30_000, 256, "sines")])
def test_candidate_set_equals_the_oracle_lb_filter(N, n, kind):
    """The scan's candidate set, element by element, against the oracle's fp64 LB filter (C6,
    P:273-276): {pos outside the window : LB^2_fp64(pos) <= T}, with T = bsf0^2 (1 + delta) the
    threshold of the GPU's window BSF (R8). The only tolerance is the fp32 summation band around
    T (|LB^2 / T - 1| <= 1e-5): a position there may go either way. The leaf-pruned scan (R11)
    and the flat ParIS scan keep the same set."""
    wl = small_workload(N, n, kind, Q=12, q_noisy=4 if kind == "walk" else 12, sigma=0.1)
    x = datagen.series(wl, 0, N)
    q, _ = datagen.queries(wl)
    qh = q.cpu().numpy()
    # one round per query (no first band, R15): the list is then the whole LB filter of bsf0
    with _build(x, first_band=-1) as ix, _build(x, flags=1, first_band=-1) as flat:
        ids, dist = ix.nn1(q)
        st = ix.stats()
        cands = [np.sort(ix.candidates(i)) for i in range(len(qh))]
        ids_f, dist_f = flat.nn1(q)
        st_f = flat.stats()
        cands_f = [np.sort(flat.candidates(i)) for i in range(len(qh))]
        ex = ix.export(0, N, sax=True, perm=True)
    np.testing.assert_array_equal(ids.cpu().numpy(), ids_f.cpu().numpy())
    np.testing.assert_array_equal(dist.cpu().numpy(), dist_f.cpu().numpy())
    onepd = np.float32(1 + 2.0**-12)
    _, _, _, qm, _ = clib.summarise(qh)
    words_sorted = ex["sax"][ex["perm"]]
    checked = 0
    for i in range(len(qh)):
        assert st["rounds"][i] == 1
        np.testing.assert_array_equal(cands[i], cands_f[i])
        assert len(np.unique(cands[i])) == len(cands[i])
        T = float(np.float32(st["bsf0_d2"][i]) * onepd)
        w0, w1 = st["window"][2 * i], st["window"][2 * i + 1]
        lb_or = ref.lb2(qm[i], words_sorted, n)
        lb_or[w0:w1] = np.inf
        got = np.zeros(N, bool)
        got[cands[i]] = True
        sure = lb_or <= T * (1 - 1e-5)
        maybe = lb_or <= T * (1 + 1e-5)
        assert got[sure].all(), f"query {i}: {int((sure & ~got).sum())} oracle candidates missing"
        assert not (got & ~maybe).any(), f"query {i}: {int((got & ~maybe).sum())} extra candidates"
        assert st["candidates"][i] == len(cands[i])
        checked += int(sure.sum())
        assert st["leaves_alive"][i] <= (N + st["leaf_size"] - 1) // st["leaf_size"]
    assert checked > 0
    assert st_f["leaves_alive"] == [0] * len(qh)


def test_ties_duplicates_constants_and_exact_copies():
    N, n = 5_000, 256
    wl = small_workload(N, n, Q=8)
    x = datagen.series(wl, 0, N).clone()
    x[4000] = x[17]  # exact duplicate: the tie must resolve to id 17
    x[4001] = x[17] * 3.0 + 2.0  # same shape after z-norm (up to rounding)
    x[10] = 1.5  # constant series -> all-zero row
    x[4002] = -7.0
    q, _ = datagen.queries(wl)
    q = q.clone()
    q[0] = x[4000]
    q[1] = x[10] + 1.0  # constant query -> the all-zero row; ties between ids 10 and 4002 -> 10
    q[2] = x[123]
    xh, qh = x.cpu().numpy(), q.cpu().numpy()
    ids_or, dist_or, _ = oracle_nn1(xh, qh)
    with _build(x) as ix:
        ids, dist = ix.nn1(q)
    ids, dist = ids.cpu().numpy(), dist.cpu().numpy()
    assert_nn_parity(ids, dist, ids_or, dist_or)
    assert ids[0] == 17 and dist[0] == 0.0
    assert ids[1] == 10 and dist[1] == 0.0
    assert ids[2] == 123 and dist[2] == 0.0


@pytest.mark.parametrize("opts", [dict(window_L=1), dict(window_L=4096), dict(cand_cap=7), dict(batch_Q=3),
                                  dict(slack_log2=-20), dict(probe_bits=0xFFFFFFFF), dict(probe_bits=5, probe_L=1),
                                  dict(probe_bits=2, probe_L=1024), dict(flags=1), dict(window_L=2048),
                                  dict(window_L=1024), dict(window_L=512, probe_L=64), dict(probe_L=256),
                                  dict(probe_bits=3, probe_L=512), dict(first_band=-1), dict(first_band=0.3),
                                  dict(first_band=0.02, cand_cap=7), dict(first_band=0.999)])
def test_options_do_not_change_answers(opts):
    N, n = 30_000, 256
    wl = small_workload(N, n, Q=12, q_noisy=4)
    x = datagen.series(wl, 0, N)
    q, _ = datagen.queries(wl)
    ids_or, dist_or, _ = oracle_nn1(x.cpu().numpy(), q.cpu().numpy())
    with _build(x, **opts) as ix:
        ids, dist = ix.nn1(q)
        st = ix.stats()
    assert_nn_parity(ids.cpu().numpy(), dist.cpu().numpy(), ids_or, dist_or)
    if "cand_cap" in opts:
        assert max(st["rounds"]) >= 2  # overflow rounds were exercised


def test_tiny_collections():
    for N in (1, 2, 3, 31, 33, 1023, 1025):
        wl = small_workload(N, 64, Q=5, seed=N)
        x = datagen.series(wl, 0, N)
        q, _ = datagen.queries(wl)
        ids_or, dist_or, _ = oracle_nn1(x.cpu().numpy(), q.cpu().numpy())
        with _build(x) as ix:
            ids, dist = ix.nn1(q)
        assert_nn_parity(ids.cpu().numpy(), dist.cpu().numpy(), ids_or, dist_or)


def test_streamed_build_equals_device_build():
    N, n = 50_000, 256
    wl = small_workload(N, n)
    x = datagen.series(wl, 0, N)
    fptr, ctx = datagen.fill_callback(wl)
    with _build(x) as a, isax.Index.build_stream(N, n, fptr, ctx, chunk=7_000) as b:
        ea = a.export(0, N, sax=True, perm=True, stored=True)
        eb = b.export(0, N, sax=True, perm=True, stored=True)
    for k in ea:
        np.testing.assert_array_equal(ea[k], eb[k])
    with isax.Index.build(x.cpu().numpy()) as c:  # host pointer -> chunked H2D path
        ec = c.export(0, N, sax=True, perm=True, stored=True)
    for k in ea:
        np.testing.assert_array_equal(ea[k], ec[k])


def test_errors():
    x = torch.zeros((10, 256), device="cuda")
    with pytest.raises(isax.IsaxError) as e:
        isax.Index.build(x[:0])
    assert e.value.name == "ISAX_E_EMPTY"
    with pytest.raises(isax.IsaxError) as e:
        isax.Index.build(torch.zeros((10, 250), device="cuda"))
    assert e.value.name == "ISAX_E_INVAL"
    with pytest.raises(isax.IsaxError) as e:
        isax.Index.build(x, card=3)
    assert e.value.name == "ISAX_E_INVAL"
    with pytest.raises(isax.IsaxError) as e:
        isax.Index.build(x, w=8)
    assert e.value.name == "ISAX_E_UNSUPPORTED"
    bad = torch.randn((100, 256), device="cuda")
    bad[37, 5] = float("nan")
    with pytest.raises(isax.IsaxError) as e:
        isax.Index.build(bad)
    assert e.value.name == "ISAX_E_NONFINITE"
    with isax.Index.build(torch.randn((100, 256), device="cuda").cumsum(1)) as ix:
        q = torch.randn((3, 256), device="cuda")
        q[1, 0] = float("inf")
        with pytest.raises(isax.IsaxError) as e:
            ix.nn1(q)
        assert e.value.name == "ISAX_E_NONFINITE"
        ids, dist = ix.nn1(torch.zeros((0, 256), device="cuda"))
        assert ids.numel() == 0


def test_heavy_overflow_rounds():
    """A poor approximate answer (one-row window, no probes) and a small candidate capacity: every
    CTA's shared buffer fills, the global lists overflow and are dropped for the round (CB_OVF),
    and the queries finish in several LB bands (R10). Answers stay exact."""
    N, n = 300_000, 128
    wl = small_workload(N, n, Q=20, q_noisy=6)
    x = datagen.series(wl, 0, N)
    q, _ = datagen.queries(wl)
    ids_or, dist_or, _ = oracle_nn1(x.cpu().numpy(), q.cpu().numpy())
    with _build(x, window_L=1, probe_bits=0xFFFFFFFF, cand_cap=1500) as ix:
        ids, dist = ix.nn1(q)
        st = ix.stats()
    assert_nn_parity(ids.cpu().numpy(), dist.cpu().numpy(), ids_or, dist_or)
    assert max(st["rounds"]) >= 3


def test_c_abi_from_plain_c(tmp_path):
    """The boundary from C: examples/nn1_c.c builds, queries through isax_nn1 (host buffers) and
    checks every answer against its own brute force."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2009_01614_b200")
    exe = str(tmp_path / "nn1_c")
    subprocess.run(["gcc", "-O2", "-std=c99", "-I", os.path.join(root, "include"), os.path.join(root, "examples", "nn1_c.c"),
                    "-L", lib, "-lisax", f"-Wl,-rpath,{lib}", "-lm", "-o", exe], check=True)
    r = subprocess.run([exe, "20000", "256", "8"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("ok")


def test_many_queries_span_batches():
    """Q = 1100 with the default batch_Q (1024): a full batch and a ragged one of 76, each with its
    own share of the candidate pool; answers equal the oracle's."""
    N, n, Q = 20_000, 128, 1100
    wl = small_workload(N, n, "sines", Q=Q, q_noisy=600, sigma=0.05)
    x = datagen.series(wl, 0, N)
    q, _ = datagen.queries(wl)
    ids_or, dist_or, _ = oracle_nn1(x.cpu().numpy(), q.cpu().numpy())
    with _build(x) as ix:
        ids, dist = ix.nn1(q)
        st = ix.stats()
    assert_nn_parity(ids.cpu().numpy(), dist.cpu().numpy(), ids_or, dist_or)
    # main window of every query: 3072 rows, or a 512-row kd cell in batches run best-first (R15)
    assert len(st["rounds"]) == Q and min(st["window_rows"]) >= min(512, N)


def test_config1_at_its_own_seeds():
    """BASELINE.json configs[0] exactly: 100,000 walks x 256 (data seed 1), 10 walk queries (seed 2)."""
    wl = datagen.WORKLOADS[1]
    x = datagen.series(wl, 0, wl.N)
    q, _ = datagen.queries(wl)
    ids_or, dist_or, _ = oracle_nn1(x.cpu().numpy(), q.cpu().numpy())
    with _build(x) as ix:
        ids, dist = ix.nn1(q)
    assert_nn_parity(ids.cpu().numpy(), dist.cpu().numpy(), ids_or, dist_or)


@pytest.mark.parametrize("opts", [dict(), dict(window_L=1, probe_bits=0xFFFFFFFF), dict(cand_cap=64)])
def test_many_exact_ties_terminate(opts):
    """More near ties than a near list holds (ties -> lowest id; R9): 300 copies of
    series 17 and 300 constant series (all z-normalise to the zero row). The lists overflow, grow
    and the queries rescan once; the answers are the lowest ids."""
    N, n = 6_000, 256
    wl = small_workload(N, n, Q=6)
    x = datagen.series(wl, 0, N).clone()
    x[1000:1300] = x[17]
    x[3000:3300] = 1.5
    q, _ = datagen.queries(wl)
    q = q.clone()
    q[0] = x[17] * 2.0 + 1.0  # the same shape after z-norm
    q[1] = -4.0  # constant query: d = 0 to every constant row
    q[2] = x[1150]
    xh, qh = x.cpu().numpy(), q.cpu().numpy()
    ids_or, dist_or, _ = oracle_nn1(xh, qh, K=1024)
    with _build(x, **opts) as ix:
        ids, dist = ix.nn1(q)
        st = ix.stats()
    ids, dist = ids.cpu().numpy(), dist.cpu().numpy()
    assert_nn_parity(ids, dist, ids_or, dist_or)
    assert ids[0] == 17 and ids[1] == 3000 and ids[2] == 17
    assert max(st["near"][:3]) > 256  # the near lists did overflow their first capacity


@pytest.mark.parametrize("exact_copy", [True, False])
def test_tiny_cand_cap_with_equal_bounds(exact_copy):
    """cand_cap = 7 and 40 identical rows sharing one LB^2 (0 for an exact-copy query): the LB
    band cannot be split, so the rounds split the sorted positions (R10). Answers exact."""
    N, n = 20_000, 128
    wl = small_workload(N, n, Q=4)
    x = datagen.series(wl, 0, N).clone()
    x[5000:5040] = x[333]
    q, _ = datagen.queries(wl)
    q = q.clone()
    q[0] = x[333] if exact_copy else x[333] + 0.05 * torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    ids_or, dist_or, _ = oracle_nn1(x.cpu().numpy(), q.cpu().numpy(), K=64)
    with _build(x, cand_cap=7, window_L=1, probe_bits=0xFFFFFFFF) as ix:
        ids, dist = ix.nn1(q)
        st = ix.stats()
    assert_nn_parity(ids.cpu().numpy(), dist.cpu().numpy(), ids_or, dist_or)
    if exact_copy:
        assert ids[0].item() == 333
    assert max(st["rounds"]) >= 3


def _gpu_fp64_d2(q, y):
    """finalize_kernel's fp64 d^2: lane l sums elements l, l + 32, ... left to right, then the
    xor butterfly (16, 8, 4, 2, 1) over the lanes."""
    q64, y64 = q.astype(np.float64), y.astype(np.float64)
    v = []
    for lane in range(32):
        acc = 0.0
        for i in range(lane, len(q), 32):
            d = q64[i] - y64[i]
            acc = acc + d * d
        v.append(acc)
    for o in (16, 8, 4, 2, 1):
        v = [v[l] + v[l ^ o] for l in range(32)]
    return v[0]


def test_finalize_is_exact_when_fp64_ties():
    """Two rows whose fp64 d^2 (the kernel's summation order) say the lower id is at least as
    near, while the exact d^2 says the higher id is nearer: the answer must be the higher id
    (lexicographic (exact d^2, id), north_star / SPEC.md:285). Built from integer raw rows (so
    z-norm of a permutation is the permutation of the z-norm, bit for bit: every fp64 sum is
    exact) and a query with two 1-ulp-apart tiny elements; searched over seeds on the host with
    the oracle's z-norm."""
    from fractions import Fraction

    n = 256
    found = None
    for seed in range(400):
        rng = np.random.default_rng(seed)
        xa = np.cumsum(rng.integers(-3, 4, n)).astype(np.float32)
        i, j = (int(v) for v in rng.choice(n, 2, replace=False))
        if xa[i] == xa[j]:
            continue
        xb = xa.copy()
        xb[i], xb[j] = xa[j], xa[i]  # d^2(q, b) - d^2(q, a) = 2 (q_i - q_j)(y_i - y_j), exactly
        ya, _, _ = ref.znorm(xa[None])
        yb, _, _ = ref.znorm(xb[None])
        # a query near row a whose normalised elements i, j are tiny and 1 ulp apart: the other
        # elements are centred (mean ~1e-9), then q_i = fp32(mean), q_j the next fp32 up
        qr = (ya[0] + rng.standard_normal(n).astype(np.float32) * np.float32(0.01)).astype(np.float32)
        qr[i] = qr[j] = 0
        rest = np.ones(n, bool)
        rest[[i, j]] = False
        for _ in range(4):
            qr[rest] = (qr[rest] - np.float32(qr.astype(np.float64).sum() / (n - 2))).astype(np.float32)
        qr[i] = np.float32(qr.astype(np.float64).sum() / n)
        qr[j] = np.nextafter(qr[i], np.float32(1))
        qy, _, _ = ref.znorm(qr[None])
        ea, eb = ref.ed2_exact(qy[0], ya[0]), ref.ed2_exact(qy[0], yb[0])
        fa, fb = _gpu_fp64_d2(qy[0], ya[0]), _gpu_fp64_d2(qy[0], yb[0])
        if ea > eb and fa <= fb:  # the fp64 rule would pick row a (lower id); the exact one b
            found = (xa, xb, qr, ea, eb)
            break
        if eb > ea and fb <= fa:
            found = (xb, xa, qr, eb, ea)
            break
    assert found is not None, "no fp64-tie construction found"
    xa, xb, qr, ea, eb = found
    N = 4_000
    wl = small_workload(N, n, Q=2)
    x = datagen.series(wl, 0, N).clone()
    x[100] = torch.from_numpy(xa).cuda()  # the lower id: exactly farther
    x[2500] = torch.from_numpy(xb).cuda()
    q, _ = datagen.queries(wl)
    q = q.clone()
    q[0] = torch.from_numpy(qr).cuda()
    ids_or, dist_or, d2_or = oracle_nn1(x.cpu().numpy(), q.cpu().numpy())
    assert ids_or[0] == 2500 and d2_or[0] == eb and Fraction(ea) > Fraction(eb)
    with _build(x) as ix:
        ids, dist = ix.nn1(q)
    assert_nn_parity(ids.cpu().numpy(), dist.cpu().numpy(), ids_or, dist_or)


def test_stats_report_build_stages_and_scan_counters():
    """isax_stats: the build's stage times are there right after the build, and after a call the
    scan's own counters are consistent: every lookup belongs to a node or member bound (16 each),
    and every bound read a summary (32 B) or a word (16 B)."""
    N, n = 60_000, 256
    wl = small_workload(N, n, Q=20)
    x = datagen.series(wl, 0, N)
    q, _ = datagen.queries(wl)
    with _build(x, first_band=-1) as ix:
        st0 = ix.stats()
        assert all(st0["build_ms"][k] > 0 for k in ("summarise", "sort", "kd_and_node_summaries", "permute"))
        ix.nn1(q)
        st = ix.stats()
    lk, by = st["scan_lookups_first_launch"], st["scan_bytes_first_launch"]
    assert lk > 0 and lk % 16 == 0
    tests = lk // 16
    # between all-member (16 B each) and all-node (32 B each) tests, plus 5 B per candidate
    assert 16 * tests <= by <= 32 * tests + 5 * sum(st["candidates"]) + 64
    assert st["cell_size"] == 8 and st["leaf_size"] == 32
    assert st["leaf_pairs_first_launch"] == sum(st["leaves_alive"])


def test_save_load_round_trip(tmp_path):
    """isax_save / isax_load: the loaded index holds the same words, permutation and rows, and
    returns the same (oracle-checked) answers; bad files give the documented errors."""
    N, n = 40_000, 128
    wl = small_workload(N, n, Q=12, q_noisy=4)
    x = datagen.series(wl, 0, N)
    q, _ = datagen.queries(wl)
    ids_or, dist_or, _ = oracle_nn1(x.cpu().numpy(), q.cpu().numpy())
    path = str(tmp_path / "ix.isax")
    with _build(x) as ix:
        ids0, dist0 = ix.nn1(q)
        ex0 = ix.export(0, N, sax=True, perm=True, stored=True)
        ix.save(path)
    assert os.path.getsize(path) > N * n * 4
    with isax.Index.load(path) as ix2:
        assert (ix2.N, ix2.n, ix2.w, ix2.card) == (N, n, 16, 256)
        ex1 = ix2.export(0, N, sax=True, perm=True, stored=True)
        ids1, dist1 = ix2.nn1(q)
    for k in ("sax", "perm", "stored"):
        np.testing.assert_array_equal(ex0[k], ex1[k])
    assert_nn_parity(ids1.cpu().numpy(), dist1.cpu().numpy(), ids_or, dist_or)
    np.testing.assert_array_equal(ids0.cpu().numpy(), ids1.cpu().numpy())
    np.testing.assert_array_equal(dist0.cpu().numpy(), dist1.cpu().numpy())
    # a truncated file, a file that is not an index, a missing file
    blob = open(path, "rb").read()
    bad = str(tmp_path / "short.isax")
    open(bad, "wb").write(blob[: len(blob) // 2])
    with pytest.raises(isax.IsaxError) as e:
        isax.Index.load(bad)
    assert e.value.name == "ISAX_E_IO"
    open(bad, "wb").write(b"not an index" * 20)
    with pytest.raises(isax.IsaxError) as e:
        isax.Index.load(bad)
    assert e.value.name == "ISAX_E_INVAL"
    with pytest.raises(isax.IsaxError) as e:
        isax.Index.load(str(tmp_path / "missing.isax"))
    assert e.value.name == "ISAX_E_IO"


def test_summaries_bit_exact_when_the_row_sum_rounds():
    """Rows whose fp64 sum rounds (a value next to zero, a denormal, a wide dynamic range) depend on
    the summation order: the kernel must take the definition's left-to-right order (R3) and give
    the oracle's words and rows bit for bit; all-zero and nearly-zero rows too."""
    N, n = 4_096, 256
    wl = small_workload(N, n, "walk")
    x = datagen.series(wl, 0, N).clone()
    x[5, 17] = 1e-12          # 2^-40 of the row's magnitude: the sum rounds
    x[6, 3] = 1e-40           # a denormal
    x[7, :] = 0.0
    x[7, 100] = 3.0           # zeros and one value: exact
    x[8, 0] = 1e20            # wide dynamic range
    x[8, 1] = 1e-3
    x[9, :] = 0.0             # all zeros -> the all-zero row
    x[10, :] = x[10, :] * 1e-30  # small normal values
    x[11, ::2] = 1.00000012   # neighbours one ulp apart
    x[11, 1::2] = 1.0
    for r in range(40, 60):    # a value next to zero at every quarter boundary and inside
        x[r, (r - 40) * 13 % n] = 3e-9
    xh = x.cpu().numpy()
    with _build(x) as ix:
        ex = ix.export(0, N, sax=True, perm=True, stored=True)
    y, mu, sd, m, word = clib.summarise(xh)
    np.testing.assert_array_equal(ex["sax"], word)
    np.testing.assert_array_equal(ex["stored"], y[ex["perm"].astype(np.int64)])
