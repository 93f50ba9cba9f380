// api.cu: the C-ABI entry points of libisax.so (include/isax.h).
//
// This is host orchestration only: argument checks, pointer-kind detection, device memory,
// the build's two passes, and the query batches and rounds. Every step of the method runs in
// the kernels of summarise.cu, sort.cu, permute.cu, query.cu, lbscan.cu and refine.cu. There
// is no CPU fallback: without a usable CUDA device every call returns ISAX_E_CUDA.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>

#include <nvtx3/nvToolsExt.h>  // header-only; ranges show up under nsys / ncu --nvtx, no-ops otherwise

#include "isax_internal.cuh"
#include "round_plan.h"

namespace {
struct NvtxRange {  // an NVTX range for the enclosing scope
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};
}  // namespace

namespace isax {

static thread_local std::string g_err;

int set_error(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

int cuda_error(cudaError_t e, const char *what) {
    std::string m = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    if (e == cudaErrorMemoryAllocation) return set_error(ISAX_E_NOMEM, m);
    return set_error(ISAX_E_CUDA, m);
}

static bool is_device_ptr(const void *p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Every entry point that touches an index runs on the index's device (a caller may
// have another device current); the caller's current device is restored on return.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
            return;
        }
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

static isax_opts default_opts(const isax_opts *o) {
    isax_opts r{3072, -12, 1024, 0, 0, 5, 128, 0.f};  // cand_cap 0: chosen per batch (alloc_scratch, nn1_device)
    if (o) {
        if (o->probe_bits) r.probe_bits = o->probe_bits;
        if (o->probe_L) r.probe_L = o->probe_L;
        if (o->window_L) r.window_L = o->window_L;
        if (o->slack_log2) r.slack_log2 = o->slack_log2;
        if (o->batch_Q) r.batch_Q = o->batch_Q;
        if (o->cand_cap) r.cand_cap = o->cand_cap;
        r.first_band = o->first_band;
        r.flags = o->flags;
    }
    return r;
}

static int check_geometry(uint64_t N, uint32_t n, uint32_t w, uint32_t card, const isax_opts &o) {
    if (w == 0 || n == 0) return set_error(ISAX_E_INVAL, "n and w must be positive");
    if (n % w) return set_error(ISAX_E_INVAL, "w must divide n (S:71)");
    if (card < 2 || card > 256 || (card & (card - 1))) return set_error(ISAX_E_INVAL, "card must be a power of two in [2, 256]");
    if (N == 0) return set_error(ISAX_E_EMPTY, "empty collection (N == 0)");
    if (w != 16 || card != 256) return set_error(ISAX_E_UNSUPPORTED, "v1 supports w=16, card=256 only");
    if (n % 64 || n > 1024) return set_error(ISAX_E_UNSUPPORTED, "v1 supports n a multiple of 64 in [64, 1024]");
    if (N >= 0xffffffffull) return set_error(ISAX_E_UNSUPPORTED, "v1 supports N < 2^32 - 1");
    if (o.window_L == 0 || o.window_L > 4096) return set_error(ISAX_E_INVAL, "window_L must be in [1, 4096]");
    if (o.slack_log2 > -8 || o.slack_log2 < -20) return set_error(ISAX_E_INVAL, "slack_log2 must be in [-20, -8]");
    if (o.batch_Q > 1024) return set_error(ISAX_E_INVAL, "batch_Q must be <= 1024");
    if (o.flags & ~ISAX_FLAG_FLAT_SCAN) return set_error(ISAX_E_INVAL, "unknown flags");
    if (o.probe_bits != ISAX_PROBES_NONE && o.probe_bits > 5) return set_error(ISAX_E_INVAL, "probe_bits must be <= 5");
    if (o.probe_L == 0 || o.probe_L > 1024) return set_error(ISAX_E_INVAL, "probe_L must be in [1, 1024]");
    if (!(o.first_band < 1.0f) || o.first_band != o.first_band) return set_error(ISAX_E_INVAL, "first_band must be < 1");
    return ISAX_OK;
}

template <class T>
static cudaError_t dmalloc(T **p, size_t count, size_t *acc) {
    cudaError_t e = cudaMalloc((void **)p, std::max<size_t>(count, 1) * sizeof(T));
    if (e == cudaSuccess && acc) *acc += std::max<size_t>(count, 1) * sizeof(T);
    return e;
}

static void free_scratch(isax_index *ix) {
    QueryScratch &q = ix->qs;
    cudaFree(q.qy); cudaFree(q.qpaa); cudaFree(q.qsax); cudaFree(q.lut); cudaFree(q.lut8); cudaFree(q.lut8c); cudaFree(q.qconst); cudaFree(q.pwin);
    cudaFree(q.cand); cudaFree(q.candq); cudaFree(q.cand2); cudaFree(q.candq2); cudaFree(q.cnt_f); cudaFree(q.qscale); cudaFree(q.qT);
    cudaFree(q.near); cudaFree(q.near_off); cudaFree(q.near_cap);
    cudaFree(q.qmap); cudaFree(q.qband); cudaFree(q.cand_hist); cudaFree(q.task_ctr); cudaFree(q.qmap2); cudaFree(q.scan_entries); cudaFree(q.scan_ctl); cudaFree(q.qkept);
    cudaFree(q.status);  // bsf, bsf_scan, cand_cnt, cand_cnt2, cnt_hi, near_cnt, flag, counters, win, leaves, byte counters
    if (q.h_mirror) cudaFreeHost(q.h_mirror);
    q = QueryScratch{};
}

// Candidate lists. With opts.cand_cap set, every query of a batch gets that capacity. By default
// the lists share one pool of CAND_POOL entries (about 12 B each), split evenly over the queries of
// each batch: a batch of B queries gets min(N, 2^23, pool / B) per query (nn1_device). The pool is
// halved while the scratch does not fit in device memory (down to 2^16 per query slot). A query
// that overflows its capacity runs more rounds (R10), each a rescan, refining its smallest bounds
// first. Small batches of random-walk queries (100 over 200M series: a few keep millions of
// candidates) get the generous 2^23; a batch of 1000 near-duplicate queries gets 2^20, where the
// smallest-bounds-first rounds skip most of a heavy query's candidates (BASELINE config 5).
constexpr uint64_t CAND_POOL = 1ull << 30;
constexpr float FB_FRAC = 0.02f;      // R15: the adaptive first band's fraction of the window threshold
constexpr uint32_t FB_REPROBE = 512;  // longest run in the preferred mode before the other one is re-timed
constexpr uint32_t PROBE_L_BEST = 64; // probe window rows in best-first mode (the probes only seed the band)
constexpr uint32_t WIN_L_BEST = 512;  // main window rows in best-first mode
static int alloc_scratch_cap(isax_index *ix, uint32_t cap);
static int alloc_scratch(isax_index *ix) {
    if (ix->qs.cap_Q) return ISAX_OK;
    if (ix->opts.cand_cap) return alloc_scratch_cap(ix, ix->opts.cand_cap);
    const uint64_t per_max = std::min<uint64_t>(ix->N, 1ull << 23);
    uint32_t cap = (uint32_t)std::min<uint64_t>(per_max, std::max<uint64_t>(CAND_POOL / ix->opts.batch_Q, 1));
    for (;;) {
        const int rc = alloc_scratch_cap(ix, cap);
        if (rc != ISAX_E_NOMEM || cap <= (1u << 16)) return rc;
        cap = std::max(cap / 2, 1u << 16);
    }
}

static int alloc_scratch_cap(isax_index *ix, uint32_t cap) {
    QueryScratch &q = ix->qs;
    const uint32_t Q = ix->opts.batch_Q;
    size_t acc = 0;
    cudaError_t e = cudaSuccess;
#define A(ptr, cnt) \
    if (e == cudaSuccess) e = dmalloc(&q.ptr, (size_t)(cnt), &acc)
    A(qy, (size_t)Q * ix->n);
    A(qpaa, (size_t)Q * W);
    A(qsax, (size_t)Q * W);
    A(lut, (size_t)Q * W * CARD);
    A(lut8, (size_t)Q * W * CARD);
    A(lut8c, (size_t)Q * (W / 2) * CARD);
    A(qconst, 2 * (size_t)Q);
    A(pwin, (size_t)Q * MAX_PROBES);
    A(cand, (size_t)Q * cap);
    A(candq, (size_t)Q * cap);
    A(cand2, (size_t)Q * cap);
    A(candq2, (size_t)Q * cap);
    A(cnt_f, Q);
    A(qscale, Q);
    A(qT, Q);
    A(near, (size_t)Q * NEAR_K);
    A(near_off, Q);
    A(near_cap, Q);
    A(qmap, Q);
    A(qband, Q);
    A(cand_hist, (size_t)Q * HIST_BINS);
    A(task_ctr, 1);
    q.scan_groups = (Q + 15) / 16 + 1;  // (a batch of 2-15 queries scans in two groups of 1-8)
    A(scan_entries, (size_t)q.scan_groups * ((ix->N + SUPER_SIZE - 1) / SUPER_SIZE));
    A(scan_ctl, 4 * (size_t)q.scan_groups);
    A(qkept, Q);
    A(qmap2, Q);
#undef A
    if (e == cudaSuccess) {
        e = cudaMalloc(&q.status, StatusBlock::bytes(Q));
        if (e == cudaSuccess) {
            acc += StatusBlock::bytes(Q);
            StatusBlock sb;
            sb.carve(q.status, Q);
            q.bsf = sb.bsf;
            q.bsf_scan = sb.bsf_scan;
            q.scan_bytes_dev = sb.scan_bytes_dev;
            q.refine_bytes = sb.refine_bytes;
            q.cand_cnt = sb.cand_cnt;
            q.cand_cnt2 = sb.cand_cnt2;
            q.cnt_hi = sb.cnt_hi;
            q.near_cnt = sb.near_cnt;
            q.flag = sb.flag;
            q.counters = sb.counters;
            q.win = sb.win;
            q.counters_leaf = sb.leaves;
        }
    }
    if (e == cudaSuccess) e = cudaMallocHost(&q.h_mirror, HostMirror::bytes(Q));
    if (e == cudaSuccess) q.hm.carve(q.h_mirror, Q);
    if (e != cudaSuccess) {
        free_scratch(ix);
        cudaGetLastError();  // clear a sticky allocation error before a smaller retry
        if (e == cudaErrorMemoryAllocation) return set_error(ISAX_E_NOMEM, "query scratch does not fit in device memory");
        return cuda_error(e, "allocating query scratch");
    }
    q.cap_Q = Q;
    q.near_pool = (uint64_t)Q * NEAR_K;
    q.cand_cap = q.cand_cap_slot = cap;
    ix->device_bytes += acc;
    return ISAX_OK;
}

// ------------------------------------------------------------------------------------ build
struct Source {  // where pass 1 / pass 2 read raw rows from
    const float *dev = nullptr;  // whole collection resident on the device
    const float *host = nullptr; // whole collection in host memory (chunked H2D)
    isax_fill_fn fill = nullptr; // user producer (chunked)
    void *ctx = nullptr;
};

static int build_impl(const Source &src, uint64_t N, uint32_t n, uint32_t w, uint32_t card, uint64_t chunk,
                      const isax_opts *opts, isax_index **out) {
    if (!out) return set_error(ISAX_E_INVAL, "out is NULL");
    isax_opts o = default_opts(opts);
    int rc = check_geometry(N, n, w, card, o);
    if (rc) return rc;
    int dev = 0;
    ISAX_CUDA(cudaGetDevice(&dev));
    cudaStream_t s;
    ISAX_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    isax_index *ix = new isax_index();
    ix->N = N; ix->n = n; ix->w = w; ix->card = card; ix->opts = o; ix->device = dev;
    ix->win_auto = !(opts && opts->window_L);
    ix->win_L = o.window_L;
    ix->pr_auto = !(opts && opts->probe_L);
    ix->pr_L = o.probe_L;
    uint8_t *sax_by_id = nullptr;
    uint4 *keys = nullptr;
    double2 *musig = nullptr;
    uint32_t *ids = nullptr, *bad = nullptr, *inv = nullptr;
    float *stage = nullptr;
    uint32_t h_bad = 0;
    const bool chunked = src.dev == nullptr;
    if (chunk == 0) chunk = std::max<uint64_t>(1, (1ull << 30) / ((uint64_t)n * 4));  // ~1 GB per chunk
    chunk = std::min(chunk, N);
    cudaError_t e = cudaSuccess;
    // stage timing (isax_stats "build_ms"): event pairs around the stage's launches, read at the end
    std::vector<cudaEvent_t> tev[4];  // 0 summarise, 1 sort, 2 kd order + node summaries, 3 permute
    auto tick = [&](int stage) {
        cudaEvent_t e = nullptr;
        if (cudaEventCreate(&e) == cudaSuccess) {
            cudaEventRecord(e, s);
            tev[stage].push_back(e);
        }
    };
    auto fail = [&](int code) {
        cudaStreamSynchronize(s);
        for (auto &v : tev)
            for (cudaEvent_t e : v) cudaEventDestroy(e);
        cudaFree(sax_by_id); cudaFree(keys); cudaFree(musig); cudaFree(ids); cudaFree(bad); cudaFree(inv);
        cudaFree(stage);
        cudaFree(ix->stored); cudaFree(ix->sax); cudaFree(ix->perm); cudaFree(ix->lmeta); cudaFree(ix->cmeta); cudaFree(ix->smeta); cudaFree(ix->hmeta);
        cudaFree(ix->skey); cudaFree(ix->ksplit);
        delete ix;
        cudaStreamDestroy(s);
        return code;
    };
#define TRY(call)                                                \
    do {                                                         \
        e = (call);                                              \
        if (e != cudaSuccess) return fail(cuda_error(e, #call)); \
    } while (0)
    TRY(dmalloc(&sax_by_id, N * W, nullptr));
    TRY(dmalloc(&keys, N, nullptr));
    TRY(dmalloc(&musig, N, nullptr));
    TRY(dmalloc(&ids, N, nullptr));
    TRY(dmalloc(&ix->perm, N, &ix->device_bytes));
    TRY(dmalloc(&bad, 1, nullptr));
    TRY(cudaMemsetAsync(bad, 0, sizeof(uint32_t), s));
    if (chunked) TRY(dmalloc(&stage, chunk * n, nullptr));
    NvtxRange nvtx_build("isax_build");
    // pass 1: summarise
    auto produce = [&](uint64_t id0, uint64_t cnt) -> int {
        if (src.host) {
            e = cudaMemcpyAsync(stage, src.host + id0 * n, cnt * n * sizeof(float), cudaMemcpyHostToDevice, s);
            if (e != cudaSuccess) return cuda_error(e, "H2D chunk");
            return ISAX_OK;
        }
        if (src.fill(src.ctx, id0, cnt, stage, (void *)s) != 0)
            return set_error(ISAX_E_CALLBACK, "fill callback returned non-zero");
        return ISAX_OK;
    };
    if (!chunked) {
        tick(0);
        launch_summarise(src.dev, N, n, 0, sax_by_id, keys, musig, bad, s);
        tick(0);
    } else {
        for (uint64_t id0 = 0; id0 < N; id0 += chunk) {
            const uint64_t cnt = std::min(chunk, N - id0);
            if ((rc = produce(id0, cnt))) return fail(rc);
            tick(0);
            launch_summarise(stage, cnt, n, id0, sax_by_id, keys, musig, bad, s);
            tick(0);
        }
    }
    TRY(cudaGetLastError());
    TRY(cudaMemcpyAsync(&h_bad, bad, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    TRY(cudaStreamSynchronize(s));
    if (h_bad) return fail(set_error(ISAX_E_NONFINITE, "a series holds NaN or Inf"));
    // canonical order (R6)
    tick(1);
    if ((rc = radix_sort_keys(keys, ids, N, ix->perm, s))) return fail(rc);
    tick(1);
    cudaFree(keys);
    keys = nullptr;
    cudaFree(ids);
    ids = nullptr;
    // padded to whole leaves: the leaf scan loads a partial last leaf's words unconditionally
    // (the padding is never a candidate: positions >= N are rejected before any emit)
    const uint64_t npad = ((N + LEAF_SIZE - 1) / LEAF_SIZE) * LEAF_SIZE;
    TRY(dmalloc(&ix->sax, npad * W, &ix->device_bytes));
    TRY(cudaMemsetAsync(ix->sax + N * W, 0xFF, (npad - N) * W, s));
    launch_gather_sax(sax_by_id, ix->perm, N, ix->sax, s);
    // kd order inside each super-node (R6b): before the node summaries and the rows
    TRY(dmalloc(&ix->skey, (N + SUPER_SIZE - 1) / SUPER_SIZE, &ix->device_bytes));
    TRY(dmalloc(&ix->ksplit, (N + SUPER_SIZE - 1) / SUPER_SIZE, &ix->device_bytes));
    tick(2);
    launch_superkd(ix->sax, ix->perm, N, ix->skey, ix->ksplit, s);
    TRY(dmalloc(&ix->lmeta, ((N + LEAF_SIZE - 1) / LEAF_SIZE) * 32, &ix->device_bytes));
    TRY(dmalloc(&ix->cmeta, (npad / KD_CELL) * 32, &ix->device_bytes));
    TRY(dmalloc(&ix->smeta, ((N + SUPER_SIZE - 1) / SUPER_SIZE) * 32, &ix->device_bytes));
    TRY(dmalloc(&ix->hmeta, ((N + HYPER_SIZE - 1) / HYPER_SIZE) * 32, &ix->device_bytes));
    launch_leaf_meta(ix->sax, N, ix->cmeta, ix->lmeta, ix->smeta, ix->hmeta, s);
    tick(2);
    TRY(cudaStreamSynchronize(s));
    cudaFree(sax_by_id);
    sax_by_id = nullptr;
    // pass 2: store the z-normalised rows in sorted order
    TRY(dmalloc(&ix->stored, N * n, &ix->device_bytes));
    if (!chunked) {
        tick(3);
        launch_gather_rows(src.dev, musig, ix->perm, N, n, ix->stored, s);
        tick(3);
    } else {
        TRY(dmalloc(&inv, N, nullptr));
        launch_invert_perm(ix->perm, N, inv, s);
        for (uint64_t id0 = 0; id0 < N; id0 += chunk) {
            const uint64_t cnt = std::min(chunk, N - id0);
            if ((rc = produce(id0, cnt))) return fail(rc);
            tick(3);
            launch_scatter_rows(stage, cnt, id0, musig, inv, n, ix->stored, s);
            tick(3);
        }
    }
    TRY(cudaGetLastError());
    TRY(cudaStreamSynchronize(s));
    cudaFree(musig); cudaFree(inv); cudaFree(stage); cudaFree(bad);
    for (int k = 0; k < 4; k++) {
        float tot = 0.f;
        for (size_t i = 0; i + 1 < tev[k].size(); i += 2) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, tev[k][i], tev[k][i + 1]) == cudaSuccess) tot += ms;
        }
        ix->st_build_ms[k] = tot;
        for (cudaEvent_t e : tev[k]) cudaEventDestroy(e);
    }
    for (auto &ev : ix->ev) TRY(cudaEventCreate(&ev));
#undef TRY
    cudaStreamDestroy(s);
    *out = ix;
    return ISAX_OK;
}

// ------------------------------------------------------------------------------------ query
static float bsf_d2_host(unsigned long long p) {
    const uint32_t hi = (uint32_t)(p >> 32);
    float f;
    memcpy(&f, &hi, 4);
    return f;
}

// Grow query i's near list after it overflowed (R9): a fresh region of the pool with room for
// twice the appends it saw. Its rescan collects every near tie of its current BSF again: those rows
// were all appended before (the BSF only falls, and a row within (1 + delta) of it completes and
// is appended wherever it is refined), so the list keeps growing until it holds them all and the
// rescan terminates. The pool grows (copying the live lists) when it has no room left.
static int grow_near(isax_index *ix, uint32_t i, uint32_t seen, cudaStream_t s) {
    QueryScratch &qs = ix->qs;
    HostMirror &hm = qs.hm;
    const uint64_t need = std::max<uint64_t>(2ull * seen, 2ull * hm.near_cap[i]);
    if (need > 0xffffffffull) return set_error(ISAX_E_UNSUPPORTED, "more than 2^32 near ties for one query");
    if (qs.near_used + need > qs.near_pool) {
        const uint64_t pool = std::max<uint64_t>(2 * qs.near_pool, qs.near_used + need);
        NearEntry *np = nullptr;
        cudaError_t e = cudaMalloc(&np, pool * sizeof(NearEntry));
        if (e != cudaSuccess) {
            cudaGetLastError();
            return cuda_error(e, "growing the near-tie pool");
        }
        ISAX_CUDA(cudaMemcpyAsync(np, qs.near, qs.near_used * sizeof(NearEntry), cudaMemcpyDeviceToDevice, s));
        ISAX_CUDA(cudaStreamSynchronize(s));
        cudaFree(qs.near);
        ix->device_bytes += (pool - qs.near_pool) * sizeof(NearEntry);
        qs.near = np;
        qs.near_pool = pool;
    }
    hm.near_off[i] = qs.near_used;
    hm.near_cap[i] = (uint32_t)need;
    qs.near_used += need;
    return ISAX_OK;
}

static int nn1_device(isax_index *ix, const float *d_q, uint32_t Q, int64_t *d_id, float *d_dist, cudaStream_t s) {
    NvtxRange nvtx_call("isax_nn1");
    int rc = alloc_scratch(ix);
    if (rc) return rc;
    QueryScratch &qs = ix->qs;
    HostMirror &hm = qs.hm;
    const float delta = std::ldexp(1.0f, ix->opts.slack_log2);
    const float onepd = 1.0f + delta;
    const float INF = std::numeric_limits<float>::infinity();
    const uint32_t NP = (uint32_t)ix->N;
    ix->st_win.assign(2 * (size_t)Q, 0);
    ix->st_cand.assign(Q, 0);
    ix->st_refined.assign(Q, 0);
    ix->st_abandoned.assign(Q, 0);
    ix->st_skipped.assign(Q, 0);
    ix->st_winrows.assign(Q, 0);
    ix->st_rounds.assign(Q, 0);
    ix->st_near.assign(Q, 0);
    ix->st_leaves.assign(Q, 0);
    ix->st_bsf0.assign(Q, 0.f);
    ix->st_bsf_final.assign(Q, 0.f);
    ix->st_ms = StageTimes{};
    ix->st_launches = 0;
    ix->st_scan_bytes = ix->st_scan_bytes_first = 0;
    ix->st_refine_bytes_first = ix->st_refine1_bytes_first = ix->st_refine2_bytes_first = 0;
    ISAX_CUDA(cudaMemsetAsync(qs.scan_bytes_dev, 0, StatusBlock::RESET_BYTES, s));  // + refine_bytes, flag
    int result = ISAX_OK;
    for (uint32_t b0 = 0; b0 < Q && result == ISAX_OK; b0 += qs.cap_Q) {
        const uint32_t B = std::min(qs.cap_Q, Q - b0);
        // the batch's share of the candidate pool (a fixed capacity when opts.cand_cap is set)
        qs.cand_cap = ix->opts.cand_cap
                          ? qs.cand_cap_slot
                          : (uint32_t)std::min<uint64_t>(std::min<uint64_t>(ix->N, 1ull << 23),
                                                         (uint64_t)qs.cand_cap_slot * qs.cap_Q / B);
        // near lists: q * NEAR_K, NEAR_K entries each (qprep_kernel writes the same on the device)
        qs.near_used = (uint64_t)B * NEAR_K;
        for (uint32_t i = 0; i < B; i++) {
            hm.near_off[i] = (unsigned long long)i * NEAR_K;
            hm.near_cap[i] = NEAR_K;
        }
        // R15: the first band (best-first order). Adaptive by default: each mode (with
        // and without the first band) is timed on the device per query; the cheaper one runs, and
        // the other is re-timed after FB_REPROBE batches. Answers never depend on it, only the work.
        const float fopt = ix->opts.first_band;
        float band0 = 0.f;
        bool adapt = false;
        if (fopt > 0.f) {
            band0 = fopt;
        } else if (fopt == 0.f) {
            adapt = true;
            bool on;
            // the first three batches run on, off, on, and the smaller of the two "on" times is kept:
            // an index's very first batch also pays for loading its kernels
            if (ix->fb_n_on < 2 || ix->fb_n_off < 1) on = ix->fb_n_on <= ix->fb_n_off;
            else {
                on = ix->fb_ms_on <= ix->fb_ms_off;
                if (ix->fb_since >= ix->fb_every) on = !on;
            }
            band0 = on ? FB_FRAC : 0.f;
        }
        // In best-first mode the approximate answer only seeds the first band's threshold, so the
        // main window shrinks to the 512-row kd cell of the query key's super-node that the query's
        // symbols lead to (plus the neighbours' kd quarters) unless the caller fixed window_L (R5,
        // R15): config 5 968K -> 1,030K q/s against the whole super-node (256 rows: 993K)
        ix->win_L = (band0 > 0.f && ix->win_auto) ? std::min<uint32_t>(ix->opts.window_L, WIN_L_BEST) : ix->opts.window_L;
        ix->pr_L = (band0 > 0.f && ix->pr_auto) ? std::min<uint32_t>(ix->opts.probe_L, PROBE_L_BEST) : ix->opts.probe_L;
        const bool timed = b0 == 0;
        if (timed) {
            ix->st_fb_frac = band0;
            ix->st_fb_improved = 0;
            ix->st_fb_banded = 0;
        }
        cudaEventRecord(ix->ev[0], s);
        launch_qprep(ix, d_q + (uint64_t)b0 * ix->n, B, band0, s, qs.flag);
        ix->st_launches += 2;
        if (timed) cudaEventRecord(ix->ev[1], s);
        launch_window(ix, B, nullptr, delta, s);
        if (timed) cudaEventRecord(ix->ev[2], s);
        // Rounds (R10). Round 0 scans the band (-1, +inf) for every query, i.e. everything
        // under the window BSF, over all positions. If a query's candidate list overflows, its
        // band is shrunk to the largest prefix of its LB histogram that fits, so the smallest
        // bounds are refined first and the BSF tightens (MESSI's priority-queue order,
        // P:349-361). When a shrunk band completes, the next band starts where it ended; it is
        // skipped when the BSF has dropped below it. A band the histogram cannot split any
        // further (its bounds all but equal, e.g. many copies of one series) is scanned over
        // parts of the sorted positions instead: halved while it overflows, then advanced with
        // doubling length. If a query's near list overflowed, its BSF is kept, the list grows
        // (grow_near), the window is re-refined and everything is rescanned, so every near tie of
        // the final BSF is collected (R9).
        // Every round ends with one host synchronisation. The finalise kernel (for the queries
        // scanned in the round) and all counter copies are enqueued before it.
        // (round 0 covers (-1, band0 * T0] when band0 > 0; qprep_kernel writes it)
        std::vector<Band> band(B, Band{-1.0f, band0 > 0.f ? -band0 : INF, 0u, NP});
        std::vector<uint32_t> plen(B, NP);  // position mode: length of the next range
        std::vector<uint32_t> nfirst(B, 0);  // consecutive overflows whose first histogram bin alone overflowed
        std::vector<char> pending(B, 1);
        std::vector<float> bsf_h(B, INF), tused(B, -1.0f), bsf0_h(B, INF);
        std::vector<uint32_t> rewin;
        bool offs_dirty = false;
        static const uint32_t dbg_rounds = getenv("ISAX_DEBUG_ROUNDS") ? (uint32_t)atoi(getenv("ISAX_DEBUG_ROUNDS")) : 0u;
        for (uint32_t round = 0;; round++) {
            NvtxRange nvtx_round(round == 0 ? "isax_nn1: round 0 (scan, candcheck, refine)" : "isax_nn1: overflow or band round");
            uint32_t nact = 0;
            for (uint32_t i = 0; i < B; i++) {
                if (!pending[i]) continue;
                pending[i] = 0;
                hm.qmap[nact] = i;
                hm.band[nact] = band[i];
                tused[i] = std::fmin(bsf_h[i] * onepd, band[i].hi);  // round 0: set after the sync
                nact++;
            }
            if (!nact) break;
            // (scanprep_kernel zeroes the candidate counts of all B slots and the scanned queries'
            // histograms)
            if (round > 0) {
                if (offs_dirty) {
                    ISAX_CUDA(cudaMemcpyAsync(qs.near_off, hm.near_off, B * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
                    ISAX_CUDA(cudaMemcpyAsync(qs.near_cap, hm.near_cap, B * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
                    offs_dirty = false;
                }
                if (!rewin.empty()) {
                    for (uint32_t i : rewin) ISAX_CUDA(cudaMemsetAsync(qs.near_cnt + i, 0, sizeof(uint32_t), s));
                    memcpy(hm.rewin, rewin.data(), rewin.size() * sizeof(uint32_t));
                    ISAX_CUDA(cudaMemcpyAsync(qs.qmap2, hm.rewin, rewin.size() * sizeof(uint32_t),
                                              cudaMemcpyHostToDevice, s));
                    launch_window(ix, (uint32_t)rewin.size(), qs.qmap2, delta, s);
                    ix->st_launches += 1;
                    rewin.clear();
                }
                // (round 0's identity map and open bands are written by qprep_kernel)
                ISAX_CUDA(cudaMemcpyAsync(qs.qmap, hm.qmap, nact * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
                ISAX_CUDA(cudaMemcpyAsync(qs.qband, hm.band, nact * sizeof(Band), cudaMemcpyHostToDevice, s));
            }
            // (round 0 of a best-first batch: the scan itself picks the queries that get the first band)
            const bool select = round == 0 && band0 > 0.f;
            ix->st_scan_bytes += launch_lbscan(ix, nact, B, qs.qmap, qs.qband, delta, select, s);
            if (select) ix->st_launches += 2;  // (the node scan's counting pass and fbdecide_kernel)
            if (timed && round == 0) cudaEventRecord(ix->ev[6], s);
            launch_candcheck(ix, B, s);
            if (timed && round == 0) cudaEventRecord(ix->ev[3], s);
            launch_refine(ix, B, delta, s, (timed && round == 0) ? &ix->ev[8] : nullptr);
            if (timed && round == 0) cudaEventRecord(ix->ev[4], s);
            // speculative: a query scanned again in a later round is finalised again
            launch_finalize(ix, nact, qs.qmap, delta, d_id + b0, d_dist + b0, s);
            cudaEventRecord(ix->ev[7], s);  // the batch's end so far (R15 policy timing)
            // scanprep + node scan + item scan (or scanprep + flat scan), candcheck, refine + filter + refine, finalize
            ix->st_launches += ((ix->opts.flags & ISAX_FLAG_FLAT_SCAN) ? 2 : 3) + 5;
            if (timed && round == 0) cudaEventRecord(ix->ev[5], s);
            ISAX_CUDA(cudaGetLastError());
            // the whole status block in one copy (StatusBlock: bsf, counters, flags, byte counts)
            ISAX_CUDA(cudaMemcpyAsync(hm.status, qs.status, StatusBlock::bytes(qs.cap_Q), cudaMemcpyDeviceToHost, s));
            ISAX_CUDA(cudaStreamSynchronize(s));
            if (*hm.flag) {
                result = set_error(ISAX_E_NONFINITE, "a query holds NaN or Inf");
                break;
            }
            if (round == 0) {  // the window BSF: the threshold round 0 used
                for (uint32_t i = 0; i < B; i++) {
                    bsf_h[i] = bsf_d2_host(hm.bsf_scan[i]);
                    bsf0_h[i] = bsf_h[i];
                    tused[i] = bsf_h[i] * onepd;
                    if (band[i].hi < 0.f) {
                        if (hm.bsf_scan[i] & 1ull) {  // the first band's edge, as the scan computed it
                            tused[i] = tused[i] * -band[i].hi;
                            band[i].hi = tused[i];
                        } else {  // the scan gave this query its whole threshold (a cheap scan, R15)
                            band[i].hi = INF;
                        }
                    }
                }
                if (band0 > 0.f && timed) {  // stats: queries whose BSF the first band at least halved; queries that got it
                    uint32_t improved = 0, banded = 0;
                    for (uint32_t i = 0; i < B; i++) {
                        improved += bsf_d2_host(hm.bsf[i]) < 0.5f * bsf0_h[i];
                        banded += std::isfinite(band[i].hi) ? 1u : 0u;
                    }
                    ix->st_fb_improved = improved;
                    ix->st_fb_banded = banded;
                }
                if (b0 == 0) {
                    ix->st_scan_bytes_first = ix->st_scan_bytes + *hm.scan_bytes_dev;
                    ix->st_scan_lookups_first = hm.scan_bytes_dev[1];  // (the second word of the 16-byte slot)
                    ix->st_refine1_bytes_first = hm.refine_bytes[0];
                    ix->st_refine2_bytes_first = hm.refine_bytes[1];
                    ix->st_refine_bytes_first = hm.refine_bytes[0] + hm.refine_bytes[1];
                    ix->st_leaf_pairs_first = 0;
                    for (uint32_t i = 0; i < B; i++) ix->st_leaf_pairs_first += hm.leaves[i];
                    ix->st_scan_q_first = nact;
                }
            }
            bool any_ovf = false;
            for (uint32_t k = 0; k < nact; k++) any_ovf |= hm.cand_cnt[hm.qmap[k]] > qs.cand_cap;
            if (any_ovf) {  // the scanned queries' LB histograms (pinned mirror)
                ISAX_CUDA(cudaMemcpyAsync(hm.hist, qs.cand_hist, (size_t)B * HIST_BINS * sizeof(uint32_t),
                                          cudaMemcpyDeviceToHost, s));
                ISAX_CUDA(cudaStreamSynchronize(s));
            }
            for (uint32_t k = 0; k < nact; k++) {
                const uint32_t i = hm.qmap[k];
                const uint32_t cnt = hm.cand_cnt[i];
                bsf_h[i] = bsf_d2_host(hm.bsf[i]);
                ix->st_cand[b0 + i] += hm.cand_cnt2[i] + hm.cnt_hi[i];  // after the exact rule (candcheck_kernel)
                ix->st_rounds[b0 + i] = round + 1;
                RoundState st{band[i], plen[i], nfirst[i]};
                const bool near_ovf = hm.near_cnt[i] > hm.near_cap[i];
                const int act = plan_next_round(st, cnt, qs.cand_cap, hm.hist + (size_t)i * HIST_BINS, near_ovf, tused[i],
                                                bsf_h[i] * onepd, NP);
                if (dbg_rounds && round % dbg_rounds == 0 && k == 0)  // ISAX_DEBUG_ROUNDS=<every>: the plan's progress
                    fprintf(stderr, "[isax] round %u: %u active; query %u: band (%.9g, %.9g] pos [%u, %u) cnt %u cap %u tused %.9g bsf %.9g -> act %d band (%.9g, %.9g] pos [%u, %u)\n",
                            round, nact, i, band[i].lo, band[i].hi, band[i].plo, band[i].phi, cnt, qs.cand_cap, tused[i], bsf_h[i], act,
                            st.band.lo, st.band.hi, st.band.plo, st.band.phi);
                band[i] = st.band;
                plen[i] = st.plen;
                nfirst[i] = st.nfirst;
                if (act == PLAN_ERROR) return set_error(ISAX_E_CUDA, "candidate list overflow at a single position");
                if (act == PLAN_RESCAN) {  // near overflow: grow the list, start over, BSF kept (R9)
                    if ((rc = grow_near(ix, i, hm.near_cnt[i], s))) return rc;
                    offs_dirty = true;
                    rewin.push_back(i);
                }
                pending[i] = act != PLAN_DONE;
            }
            // a safety net, not a budget: a round refines at least a list's worth of a query's
            // candidates, so N / cand_cap rounds per query can be legitimate (cand_cap 5 over 220K
            // series: 119,781); the net sits well above that
            if (round > 100000ull + 8ull * ix->N / std::max<uint32_t>(qs.cand_cap, 1u)) {
                result = set_error(ISAX_E_CUDA, "candidate rounds did not converge");
                break;
            }
        }
        if (result) break;
        if (adapt) {  // R15 policy: device ms per query of this batch, in its mode
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, ix->ev[0], ix->ev[7]) == cudaSuccess) {
                const float per = ms / (float)B;
                float &slot = band0 > 0.f ? ix->fb_ms_on : ix->fb_ms_off;
                uint32_t &nmeas = band0 > 0.f ? ix->fb_n_on : ix->fb_n_off;
                const bool known = ix->fb_n_on >= 2 && ix->fb_n_off >= 1;
                const bool pref_on = ix->fb_ms_on <= ix->fb_ms_off;
                const bool preferred = known && (band0 > 0.f) == pref_on;
                slot = slot < 0.f ? per : (nmeas < 2 ? std::min(slot, per) : 0.5f * (slot + per));
                nmeas++;
                if (preferred) {
                    ix->fb_since++;
                } else {  // a re-timing: back off if the choice holds, start over if it flipped
                    ix->fb_since = 0;
                    if (known) {
                        const bool now_on = ix->fb_ms_on <= ix->fb_ms_off;
                        ix->fb_every = now_on == pref_on ? std::min<uint32_t>(2 * ix->fb_every, FB_REPROBE) : 32;
                    }
                }
            } else {
                cudaGetLastError();
            }
        }
        for (uint32_t i = 0; i < B; i++) {
            ix->st_refined[b0 + i] = hm.counters[4 * i];
            ix->st_abandoned[b0 + i] = hm.counters[4 * i + 1];
            ix->st_skipped[b0 + i] = hm.counters[4 * i + 2];
            ix->st_winrows[b0 + i] = hm.counters[4 * i + 3];
            ix->st_near[b0 + i] = hm.near_cnt[i];
            ix->st_leaves[b0 + i] = hm.leaves[i];
            ix->st_bsf0[b0 + i] = bsf0_h[i];
            ix->st_bsf_final[b0 + i] = bsf_d2_host(hm.bsf[i]);
            ix->st_win[2 * (b0 + i)] = hm.win[2 * i];
            ix->st_win[2 * (b0 + i) + 1] = hm.win[2 * i + 1];
        }
        if (timed) {
            cudaEventElapsedTime(&ix->st_ms.qprep, ix->ev[0], ix->ev[1]);
            cudaEventElapsedTime(&ix->st_ms.window, ix->ev[1], ix->ev[2]);
            cudaEventElapsedTime(&ix->st_ms.lbscan, ix->ev[2], ix->ev[6]);
            cudaEventElapsedTime(&ix->st_ms.candcheck, ix->ev[6], ix->ev[3]);
            cudaEventElapsedTime(&ix->st_ms.refine, ix->ev[3], ix->ev[4]);
            cudaEventElapsedTime(&ix->st_ms.refine1, ix->ev[3], ix->ev[8]);
            cudaEventElapsedTime(&ix->st_ms.filter, ix->ev[8], ix->ev[9]);
            cudaEventElapsedTime(&ix->st_ms.refine2, ix->ev[9], ix->ev[4]);
            float tot = 0;
            cudaEventElapsedTime(&tot, ix->ev[0], ix->ev[5]);
            ix->st_ms.finalize = tot;  // whole first round of the first batch
        }
    }
    return result;
}

#ifdef ISAX_BOUNDS
// isax_debug_bounds: one check that fails when fire != 0 (shows the mechanism traps)
__global__ void bounds_probe_kernel(int fire) { ISAX_BOUND(fire == 0); }
#endif

}  // namespace isax

using namespace isax;

// ------------------------------------------------------------------------------------ save / load
// File: a header (magic, version, geometry, the byte count of every array), then the index's
// device arrays in a fixed order. A loaded index holds byte for byte what the saved one held, so
// it answers identically. Arrays move through one pinned staging buffer in chunks.
namespace {
constexpr char SAVE_MAGIC[8] = {'I', 'S', 'A', 'X', 'B', '2', '0', '0'};
constexpr uint32_t SAVE_VERSION = 2;  // bumped with the layout (v2: kd order down to 8-row cells, cell summaries)
constexpr int SAVE_ARRAYS = 9;
struct SaveHeader {
    char magic[8];
    uint32_t version, n, w, card;
    uint64_t N;
    uint32_t leaf, cell, super_, hyper;  // node sizes the arrays were built for
    uint64_t bytes[SAVE_ARRAYS];         // stored, sax, perm, skey, ksplit, lmeta, cmeta, smeta, hmeta
};
struct ArrayRef {
    void **ptr;
    uint64_t bytes;
};
void index_arrays(isax_index *ix, ArrayRef (&a)[SAVE_ARRAYS]) {
    const uint64_t N = ix->N;
    const uint64_t nleaf = (N + LEAF_SIZE - 1) / LEAF_SIZE, npad = nleaf * LEAF_SIZE;
    const uint64_t nsuper = (N + SUPER_SIZE - 1) / SUPER_SIZE, nhyper = (N + HYPER_SIZE - 1) / HYPER_SIZE;
    a[0] = {(void **)&ix->stored, N * ix->n * sizeof(float)};
    a[1] = {(void **)&ix->sax, npad * W};
    a[2] = {(void **)&ix->perm, N * sizeof(uint32_t)};
    a[3] = {(void **)&ix->skey, nsuper * sizeof(uint4)};
    a[4] = {(void **)&ix->ksplit, nsuper * sizeof(KdSplits)};
    a[5] = {(void **)&ix->lmeta, nleaf * 32};
    a[6] = {(void **)&ix->cmeta, (npad / KD_CELL) * 32};
    a[7] = {(void **)&ix->smeta, nsuper * 32};
    a[8] = {(void **)&ix->hmeta, nhyper * 32};
}
constexpr size_t IO_CHUNK = 64u << 20;
}  // namespace

extern "C" {

int isax_save(const isax_index *cix, const char *path) {
    if (!cix || !path) return set_error(ISAX_E_INVAL, "NULL argument");
    isax_index *ix = const_cast<isax_index *>(cix);
    std::lock_guard<std::mutex> lk(ix->mu);
    DeviceGuard dg(ix->device);
    ArrayRef arr[SAVE_ARRAYS];
    index_arrays(ix, arr);
    SaveHeader h{};
    memcpy(h.magic, SAVE_MAGIC, 8);
    h.version = SAVE_VERSION;
    h.n = ix->n; h.w = ix->w; h.card = ix->card; h.N = ix->N;
    h.leaf = LEAF_SIZE; h.cell = KD_CELL; h.super_ = SUPER_SIZE; h.hyper = HYPER_SIZE;
    for (int k = 0; k < SAVE_ARRAYS; k++) h.bytes[k] = arr[k].bytes;
    FILE *f = fopen(path, "wb");
    if (!f) return set_error(ISAX_E_IO, std::string("cannot open for writing: ") + path);
    void *stage = nullptr;
    if (cudaMallocHost(&stage, IO_CHUNK) != cudaSuccess) {
        fclose(f);
        cudaGetLastError();
        return set_error(ISAX_E_NOMEM, "pinned staging buffer");
    }
    int rc = ISAX_OK;
    if (fwrite(&h, sizeof h, 1, f) != 1) rc = set_error(ISAX_E_IO, "short write (header)");
    for (int k = 0; k < SAVE_ARRAYS && !rc; k++) {
        const char *src = static_cast<const char *>(*arr[k].ptr);
        for (uint64_t off = 0; off < arr[k].bytes && !rc; off += IO_CHUNK) {
            const size_t nb = (size_t)std::min<uint64_t>(IO_CHUNK, arr[k].bytes - off);
            const cudaError_t e = cudaMemcpy(stage, src + off, nb, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) rc = cuda_error(e, "D2H (save)");
            else if (fwrite(stage, 1, nb, f) != nb) rc = set_error(ISAX_E_IO, "short write");
        }
    }
    cudaFreeHost(stage);
    if (fclose(f) != 0 && !rc) rc = set_error(ISAX_E_IO, "close failed");
    return rc;
}

int isax_load(const char *path, const isax_opts *opts, isax_index **out) {
    if (!path || !out) return set_error(ISAX_E_INVAL, "NULL argument");
    FILE *f = fopen(path, "rb");
    if (!f) return set_error(ISAX_E_IO, std::string("cannot open: ") + path);
    SaveHeader h{};
    if (fread(&h, sizeof h, 1, f) != 1 || memcmp(h.magic, SAVE_MAGIC, 8) != 0) {
        fclose(f);
        return set_error(ISAX_E_INVAL, "not an isax index file");
    }
    if (h.version != SAVE_VERSION || h.leaf != LEAF_SIZE || h.cell != KD_CELL || h.super_ != SUPER_SIZE || h.hyper != HYPER_SIZE) {
        fclose(f);
        return set_error(ISAX_E_UNSUPPORTED, "index file of another layout version");
    }
    const isax_opts o = default_opts(opts);
    int rc = check_geometry(h.N, h.n, h.w, h.card, o);
    if (rc) {
        fclose(f);
        return rc;
    }
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        fclose(f);
        return cuda_error(cudaGetLastError(), "cudaGetDevice");
    }
    isax_index *ix = new isax_index();
    ix->N = h.N; ix->n = h.n; ix->w = h.w; ix->card = h.card; ix->opts = o; ix->device = dev;
    ix->win_auto = !(opts && opts->window_L);
    ix->win_L = o.window_L;
    ix->pr_auto = !(opts && opts->probe_L);
    ix->pr_L = o.probe_L;
    ArrayRef arr[SAVE_ARRAYS];
    index_arrays(ix, arr);
    void *stage = nullptr;
    auto fail = [&](int code) {
        for (int k = 0; k < SAVE_ARRAYS; k++) cudaFree(*arr[k].ptr);
        if (stage) cudaFreeHost(stage);
        fclose(f);
        delete ix;
        cudaGetLastError();
        return code;
    };
    for (int k = 0; k < SAVE_ARRAYS; k++)
        if (h.bytes[k] != arr[k].bytes) return fail(set_error(ISAX_E_INVAL, "index file: array sizes do not match its geometry"));
    if (cudaMallocHost(&stage, IO_CHUNK) != cudaSuccess) return fail(set_error(ISAX_E_NOMEM, "pinned staging buffer"));
    for (int k = 0; k < SAVE_ARRAYS; k++) {
        if (cudaMalloc(arr[k].ptr, std::max<uint64_t>(arr[k].bytes, 1)) != cudaSuccess)
            return fail(set_error(ISAX_E_NOMEM, "device memory for the index"));
        ix->device_bytes += arr[k].bytes;
        char *dst = static_cast<char *>(*arr[k].ptr);
        for (uint64_t off = 0; off < arr[k].bytes; off += IO_CHUNK) {
            const size_t nb = (size_t)std::min<uint64_t>(IO_CHUNK, arr[k].bytes - off);
            if (fread(stage, 1, nb, f) != nb) return fail(set_error(ISAX_E_IO, "index file is truncated"));
            const cudaError_t e = cudaMemcpy(dst + off, stage, nb, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) return fail(cuda_error(e, "H2D (load)"));
        }
    }
    cudaFreeHost(stage);
    stage = nullptr;
    fclose(f);
    for (auto &ev : ix->ev)
        if (cudaEventCreate(&ev) != cudaSuccess) {
            for (int k = 0; k < SAVE_ARRAYS; k++) cudaFree(*arr[k].ptr);
            delete ix;
            return cuda_error(cudaGetLastError(), "cudaEventCreate");
        }
    *out = ix;
    return ISAX_OK;
}

}  // extern "C"

extern "C" {

int isax_build(const float *series, uint64_t N, uint32_t n, uint32_t w, uint32_t card, const isax_opts *opts,
               isax_index **out) {
    if (!series && N) return set_error(ISAX_E_INVAL, "series is NULL");
    Source src;
    if (N && is_device_ptr(series)) {
        if (reinterpret_cast<uintptr_t>(series) % 16) return set_error(ISAX_E_INVAL, "device series must be 16-byte aligned");
        src.dev = series;
    } else {
        src.host = series;
    }
    return build_impl(src, N, n, w, card, 0, opts, out);
}

int isax_build_stream(uint64_t N, uint32_t n, uint32_t w, uint32_t card, isax_fill_fn fill, void *ctx, uint64_t chunk,
                      const isax_opts *opts, isax_index **out) {
    if (!fill) return set_error(ISAX_E_INVAL, "fill is NULL");
    Source src;
    src.fill = fill;
    src.ctx = ctx;
    return build_impl(src, N, n, w, card, chunk, opts, out);
}

int isax_nn1_async(const isax_index *cix, const float *d_queries, uint32_t Q, int64_t *d_out_id, float *d_out_dist,
                   void *cuda_stream) {
    if (!cix) return set_error(ISAX_E_INVAL, "index is NULL");
    if (Q == 0) return ISAX_OK;
    if (!d_queries || !d_out_id || !d_out_dist) return set_error(ISAX_E_INVAL, "NULL pointer");
    isax_index *ix = const_cast<isax_index *>(cix);
    std::lock_guard<std::mutex> lk(ix->mu);
    DeviceGuard dg(ix->device);
    ix->st_last_Q = Q;
    return nn1_device(ix, d_queries, Q, d_out_id, d_out_dist, (cudaStream_t)cuda_stream);
}

int isax_nn1(const isax_index *cix, const float *queries, uint32_t Q, int64_t *out_id, float *out_dist) {
    if (!cix) return set_error(ISAX_E_INVAL, "index is NULL");
    if (Q == 0) return ISAX_OK;
    if (!queries || !out_id || !out_dist) return set_error(ISAX_E_INVAL, "NULL pointer");
    isax_index *ix = const_cast<isax_index *>(cix);
    std::lock_guard<std::mutex> lk(ix->mu);
    DeviceGuard dg(ix->device);
    ix->st_last_Q = Q;
    // the index keeps one stream and staging buffers for host pointers (grown on demand)
    if (!ix->io_stream) ISAX_CUDA(cudaStreamCreateWithFlags(&ix->io_stream, cudaStreamNonBlocking));
    cudaStream_t s = ix->io_stream;
    const size_t qbytes = (size_t)Q * ix->n * sizeof(float);
    const bool qdev = is_device_ptr(queries), idev = is_device_ptr(out_id), ddev = is_device_ptr(out_dist);
    if (Q > ix->io_cap) {
        cudaFree(ix->io_q);
        cudaFree(ix->io_id);
        cudaFree(ix->io_dist);
        ix->io_q = nullptr;
        ix->io_id = nullptr;
        ix->io_dist = nullptr;
        ix->io_cap = 0;
        cudaError_t e = cudaMalloc(&ix->io_q, qbytes);
        if (e == cudaSuccess) e = cudaMalloc(&ix->io_id, Q * sizeof(int64_t));
        if (e == cudaSuccess) e = cudaMalloc(&ix->io_dist, Q * sizeof(float));
        if (e != cudaSuccess) return cuda_error(e, "isax_nn1 staging");
        ix->io_cap = Q;
    }
    cudaError_t e = cudaSuccess;
    if (!qdev) e = cudaMemcpyAsync(ix->io_q, queries, qbytes, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_error(e, "isax_nn1 H2D");
    int rc = nn1_device(ix, qdev ? queries : ix->io_q, Q, idev ? out_id : ix->io_id, ddev ? out_dist : ix->io_dist, s);
    if (!rc && !idev) e = cudaMemcpyAsync(out_id, ix->io_id, Q * sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    if (!rc && e == cudaSuccess && !ddev) e = cudaMemcpyAsync(out_dist, ix->io_dist, Q * sizeof(float), cudaMemcpyDeviceToHost, s);
    if (!rc && e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (!rc && e != cudaSuccess) rc = cuda_error(e, "isax_nn1 copy-out");
    if (rc) cudaStreamSynchronize(s);
    return rc;
}

int isax_export(const isax_index *ix, uint64_t first_id, uint64_t count, uint8_t *sax_by_id, uint32_t *perm,
                float *stored) {
    if (!ix) return set_error(ISAX_E_INVAL, "index is NULL");
    if (first_id > ix->N || count > ix->N - first_id) return set_error(ISAX_E_INVAL, "range out of bounds");
    DeviceGuard dg(ix->device);
    cudaStream_t s;
    ISAX_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int rc = ISAX_OK;
    cudaError_t e = cudaSuccess;
    if (perm) e = cudaMemcpyAsync(perm, ix->perm, ix->N * sizeof(uint32_t), cudaMemcpyDefault, s);
    if (e == cudaSuccess && stored && count)
        e = cudaMemcpyAsync(stored, ix->stored + first_id * ix->n, count * ix->n * sizeof(float), cudaMemcpyDefault, s);
    if (e == cudaSuccess && sax_by_id && count) {
        uint32_t *inv = nullptr;
        uint8_t *tmp = nullptr;
        e = cudaMalloc(&inv, ix->N * sizeof(uint32_t));
        if (e == cudaSuccess) e = cudaMalloc(&tmp, count * W);
        if (e == cudaSuccess) {
            launch_invert_perm(ix->perm, ix->N, inv, s);
            launch_export_sax(ix->sax, inv, first_id, count, tmp, s);
            e = cudaMemcpyAsync(sax_by_id, tmp, count * W, cudaMemcpyDefault, s);
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        cudaFree(inv);
        cudaFree(tmp);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_error(e, "isax_export");
    cudaStreamDestroy(s);
    return rc;
}

int isax_query_debug(const isax_index *cix, const float *queries, uint32_t Q, double *q_paa, uint8_t *q_sax, float *lut,
                     uint64_t first_pos, uint64_t count, float *lb2, uint32_t *win) {
    if (!cix) return set_error(ISAX_E_INVAL, "index is NULL");
    if (!queries && Q) return set_error(ISAX_E_INVAL, "queries is NULL");
    if (lb2 && (first_pos > cix->N || count > cix->N - first_pos)) return set_error(ISAX_E_INVAL, "range out of bounds");
    isax_index *ix = const_cast<isax_index *>(cix);
    std::lock_guard<std::mutex> lk(ix->mu);
    DeviceGuard dg(ix->device);
    int rc = alloc_scratch(ix);
    if (rc) return rc;
    if (Q > ix->qs.cap_Q) return set_error(ISAX_E_INVAL, "Q exceeds batch_Q");
    if (Q == 0) return ISAX_OK;
    cudaStream_t s;
    ISAX_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const size_t qbytes = (size_t)Q * ix->n * sizeof(float);
    float *dq = nullptr, *dlb = nullptr;
    uint32_t *flag = nullptr;
    cudaError_t e = cudaMalloc(&dq, qbytes);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dq, queries, qbytes, cudaMemcpyDefault, s);
    if (e == cudaSuccess) e = cudaMalloc(&flag, sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemsetAsync(flag, 0, sizeof(uint32_t), s);
    if (e == cudaSuccess) {
        ix->win_L = ix->opts.window_L;  // (the window of a call without the first band)
        ix->pr_L = ix->opts.probe_L;
        launch_qprep(ix, dq, Q, 0.f, s, flag);
        e = cudaGetLastError();
    }
    const QueryScratch &qs = ix->qs;
    if (e == cudaSuccess && q_paa) e = cudaMemcpyAsync(q_paa, qs.qpaa, (size_t)Q * W * sizeof(double), cudaMemcpyDefault, s);
    if (e == cudaSuccess && q_sax) e = cudaMemcpyAsync(q_sax, qs.qsax, (size_t)Q * W, cudaMemcpyDefault, s);
    if (e == cudaSuccess && lut) e = cudaMemcpyAsync(lut, qs.lut, (size_t)Q * W * CARD * sizeof(float), cudaMemcpyDefault, s);
    if (e == cudaSuccess && win) e = cudaMemcpyAsync(win, qs.win, (size_t)Q * 2 * sizeof(uint32_t), cudaMemcpyDefault, s);
    if (e == cudaSuccess && lb2 && count) {
        e = cudaMalloc(&dlb, (size_t)Q * count * sizeof(float));
        if (e == cudaSuccess) {
            launch_lb_dump(ix, Q, first_pos, count, dlb, s);
            e = cudaMemcpyAsync(lb2, dlb, (size_t)Q * count * sizeof(float), cudaMemcpyDefault, s);
        }
    }
    uint32_t h_flag = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h_flag, flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    rc = e == cudaSuccess ? ISAX_OK : cuda_error(e, "isax_query_debug");
    if (!rc && h_flag) rc = set_error(ISAX_E_NONFINITE, "a query holds NaN or Inf");
    cudaStreamSynchronize(s);
    cudaFree(dq); cudaFree(dlb); cudaFree(flag);
    cudaStreamDestroy(s);
    return rc;
}

int isax_debug_candidates(const isax_index *cix, uint32_t q, uint32_t *out_pos, uint64_t cap, uint64_t *count) {
    if (!cix || !count) return set_error(ISAX_E_INVAL, "index or count is NULL");
    isax_index *ix = const_cast<isax_index *>(cix);
    std::lock_guard<std::mutex> lk(ix->mu);
    const QueryScratch &qs = ix->qs;
    if (!qs.cap_Q || ix->st_last_Q == 0 || ix->st_last_Q > qs.cap_Q || q >= ix->st_last_Q)
        return set_error(ISAX_E_INVAL, "no candidate list: q out of range, or the last call spanned several batches");
    for (uint32_t i = 0; i < ix->st_last_Q; i++)
        if (ix->st_rounds[i] != 1) return set_error(ISAX_E_INVAL, "the last call ran more than one round");
    DeviceGuard dg(ix->device);
    const uint32_t n1 = qs.hm.cand_cnt2[q], n2 = qs.hm.cnt_hi[q];
    *count = (uint64_t)n1 + n2;
    if (!out_pos || cap < *count) return ISAX_OK;
    cudaError_t e = cudaMemcpy(out_pos, qs.cand2 + (uint64_t)q * qs.cand_cap, n1 * sizeof(uint32_t), cudaMemcpyDefault);
    if (e == cudaSuccess && n2)
        e = cudaMemcpy(out_pos + n1, qs.cand2 + (uint64_t)q * qs.cand_cap + (qs.cand_cap - n2), n2 * sizeof(uint32_t),
                       cudaMemcpyDefault);
    return e == cudaSuccess ? ISAX_OK : cuda_error(e, "isax_debug_candidates");
}

int isax_debug_bounds(int fire) {
#ifdef ISAX_BOUNDS
    if (!fire) return 1;
    isax::bounds_probe_kernel<<<1, 32>>>(1);
    const cudaError_t e = cudaDeviceSynchronize();
    return e == cudaSuccess ? 1 : cuda_error(e, "isax_debug_bounds");
#else
    (void)fire;
    return 0;
#endif
}

int isax_debug_plan_round(float *band_lo_hi, uint32_t *band_pos, uint32_t *state, uint32_t cand_cnt, uint32_t cap,
                          const uint32_t *hist, int near_ovf, float tused, float bsf_lim, uint32_t N) {
    if (!band_lo_hi || !band_pos || !state || !hist) return set_error(ISAX_E_INVAL, "NULL pointer");
    RoundState st{Band{band_lo_hi[0], band_lo_hi[1], band_pos[0], band_pos[1]}, state[0], state[1]};
    const int act = plan_next_round(st, cand_cnt, cap, hist, near_ovf != 0, tused, bsf_lim, N);
    band_lo_hi[0] = st.band.lo;
    band_lo_hi[1] = st.band.hi;
    band_pos[0] = st.band.plo;
    band_pos[1] = st.band.phi;
    state[0] = st.plen;
    state[1] = st.nfirst;
    return act;
}

int isax_stats(const isax_index *cix, char *buf, size_t cap) {
    if (!cix) return set_error(ISAX_E_INVAL, "index is NULL");
    isax_index *ix = const_cast<isax_index *>(cix);
    std::lock_guard<std::mutex> lk(ix->mu);
    std::string j = "{";
    char tmp[640];
    snprintf(tmp, sizeof tmp,
             "\"N\":%llu,\"n\":%u,\"window_L\":%u,\"probe_windows\":%u,\"probe_L\":%u,\"slack_log2\":%d,\"batch_Q\":%u,\"cand_cap\":%u,"
             "\"ms_first_batch\":{\"qprep\":%.4f,\"window\":%.4f,\"lbscan\":%.4f,\"candcheck\":%.4f,\"refine\":%.4f,"
             "\"refine1\":%.4f,\"filter\":%.4f,\"refine2\":%.4f,\"total\":%.4f},",
             (unsigned long long)ix->N, ix->n, ix->win_L, window_probes(ix), ix->pr_L, ix->opts.slack_log2,
             ix->opts.batch_Q, ix->qs.cand_cap, ix->st_ms.qprep, ix->st_ms.window, ix->st_ms.lbscan, ix->st_ms.candcheck, ix->st_ms.refine,
             ix->st_ms.refine1, ix->st_ms.filter, ix->st_ms.refine2, ix->st_ms.finalize);
    j += tmp;
    auto arr = [&](const char *name, const std::vector<uint32_t> &v, bool last) {
        j += "\"";
        j += name;
        j += "\":[";
        for (size_t i = 0; i < v.size(); i++) {
            if (i) j += ",";
            j += std::to_string(v[i]);
        }
        j += last ? "]" : "],";
    };
    arr("window", ix->st_win, false);
    arr("candidates", ix->st_cand, false);
    arr("refined", ix->st_refined, false);
    arr("abandoned", ix->st_abandoned, false);
    arr("skipped", ix->st_skipped, false);
    arr("window_rows", ix->st_winrows, false);
    arr("rounds", ix->st_rounds, false);
    arr("near", ix->st_near, false);
    arr("leaves_alive", ix->st_leaves, false);
    j += "\"bsf_final_d2\":[";
    for (size_t i = 0; i < ix->st_bsf_final.size(); i++) {
        char b[32];
        snprintf(b, sizeof b, "%s%.9g", i ? "," : "", ix->st_bsf_final[i]);
        j += b;
    }
    j += "],";
    j += "\"bsf0_d2\":[";
    for (size_t i = 0; i < ix->st_bsf0.size(); i++) {
        char b[32];
        snprintf(b, sizeof b, "%s%.9g", i ? "," : "", ix->st_bsf0[i]);
        j += b;
    }
    j += "],";
    {
        char b[160];
        snprintf(b, sizeof b, "\"first_band\":%.6g,\"first_band_improved\":%u,\"first_band_queries\":%u,", ix->st_fb_frac,
                 ix->st_fb_improved, ix->st_fb_banded);
        j += b;
    }
    j += "\"launches\":" + std::to_string(ix->st_launches);
    j += ",\"scan_bytes\":" + std::to_string(ix->st_scan_bytes);
    j += ",\"scan_bytes_first_launch\":" + std::to_string(ix->st_scan_bytes_first);
    j += ",\"refine_bytes_first_launch\":" + std::to_string(ix->st_refine_bytes_first);
    j += ",\"refine1_bytes_first_launch\":" + std::to_string(ix->st_refine1_bytes_first);
    j += ",\"refine2_bytes_first_launch\":" + std::to_string(ix->st_refine2_bytes_first);
    j += ",\"leaf_pairs_first_launch\":" + std::to_string(ix->st_leaf_pairs_first);
    j += ",\"scan_lookups_first_launch\":" + std::to_string(ix->st_scan_lookups_first);
    j += ",\"cell_size\":" + std::to_string(KD_CELL);
    j += ",\"scan_queries_first_launch\":" + std::to_string(ix->st_scan_q_first);
    {
        char b[160];
        snprintf(b, sizeof b, ",\"build_ms\":{\"summarise\":%.4f,\"sort\":%.4f,\"kd_and_node_summaries\":%.4f,\"permute\":%.4f}",
                 ix->st_build_ms[0], ix->st_build_ms[1], ix->st_build_ms[2], ix->st_build_ms[3]);
        j += b;
    }
    j += ",\"leaves\":" + std::to_string((ix->N + LEAF_SIZE - 1) / LEAF_SIZE);
    j += ",\"leaf_size\":" + std::to_string(LEAF_SIZE);
    j += ",\"super_size\":" + std::to_string(SUPER_SIZE);
    j += ",\"hyper_size\":" + std::to_string(HYPER_SIZE);
    j += "}";
    if (buf && cap) {
        size_t k = std::min(cap - 1, j.size());
        memcpy(buf, j.data(), k);
        buf[k] = 0;
    }
    return (int)j.size();
}

int isax_info(const isax_index *ix, uint64_t *N, uint32_t *n, uint32_t *w, uint32_t *card, uint64_t *device_bytes) {
    if (!ix) return set_error(ISAX_E_INVAL, "index is NULL");
    if (N) *N = ix->N;
    if (n) *n = ix->n;
    if (w) *w = ix->w;
    if (card) *card = ix->card;
    if (device_bytes) *device_bytes = ix->device_bytes;
    return ISAX_OK;
}

void isax_free(isax_index *ix) {
    if (!ix) return;
    {
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        cudaFree(ix->stored);
        cudaFree(ix->sax);
        cudaFree(ix->perm);
        cudaFree(ix->lmeta);
        cudaFree(ix->cmeta);
        cudaFree(ix->smeta);
        cudaFree(ix->hmeta);
        cudaFree(ix->skey);
        cudaFree(ix->ksplit);
        free_scratch(ix);
        for (auto &ev : ix->ev)
            if (ev) cudaEventDestroy(ev);
        cudaFree(ix->io_q);
        cudaFree(ix->io_id);
        cudaFree(ix->io_dist);
        if (ix->io_stream) cudaStreamDestroy(ix->io_stream);
    }
    delete ix;
}

const char *isax_last_error(void) { return g_err.c_str(); }

const char *isax_version(void) { return "isax-b200 0.1.0 sm_100a"; }

}  // extern "C"
