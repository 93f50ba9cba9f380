// query.cu: query preparation (north_star (b) "the query's PAA") and the approximate answer
// (north_star (b) "an initial best-so-far from the leaf matching the query's iSAX word").
//
//  qprep_kernel  one CTA per query: z-norm (R2, same fp64 order as the build), PAA, SAX, key,
//                the per-segment mindist LUT, and the window position. It also resets the
//                per-query counters and the packed BSF.
//                LUT[s][c] = (n/w) * max(0, beta_c - m_s, m_s - beta_{c+1})^2 in fp64, rounded
//                DOWN to fp32 (R7), so an fp32 sum of LUT entries never
//                overestimates the fp64 bound by more than its own summation error.
//                locate: the super-node whose z-order key range holds the query key (the last
//                one whose smallest key is below it; R5, R6b). One warp runs a 32-ary search
//                over the super-nodes' smallest keys: ~4 dependent loads at N = 1e8.
//  window_kernel one CTA per query refines the L sorted rows around that position. P:271-272:
//                "the real distance between the query and the best candidate series, which is
//                in the leaf with the smallest lower bound distance"; P:341-345 for MESSI.
//                The CTA reduces the window minimum first, then appends only the near ties
//                (R9), so the near list does not fill with the whole window.
#include "isax_device.cuh"

namespace isax {

#include "breakpoints.inc"

__constant__ double c_beta_q[ISAX_NBETA] = ISAX_BETA_INIT;

// The main window covers whole super-nodes around the query key's (R5, R6b). With window_L <
// 3072 the two neighbouring super-nodes are covered by their kd-descended quarters instead (two
// extra probe-sized windows), when the probe table has room for them.
__host__ __device__ __forceinline__ uint32_t neighbour_windows(uint32_t L, uint32_t P) {
    return (L < 3 * SUPER_SIZE && (1u << P) + 1 <= MAX_PROBES - 1) ? 2u : 0u;
}


// centre of the kd cell of super-node sb (depth levels down, R6b) that the symbols sy fall in; the
// super-node's centre when it has no kd splits (the partial last one)
__device__ __forceinline__ uint64_t kd_cell_centre(const KdSplits *__restrict__ ksplit, uint64_t sb, const uint32_t *sy,
                                                   uint32_t depth) {
    KdSplits ks;
    const uint4 *src = reinterpret_cast<const uint4 *>(ksplit + sb);
    uint4 *dst = reinterpret_cast<uint4 *>(&ks);
    dst[0] = __ldg(src);
    dst[1] = __ldg(src + 1);
    if (ks.s[15] == KD_NONE || depth == 0) return sb * SUPER_SIZE + SUPER_SIZE / 2;
    uint32_t node = 0;
    for (uint32_t lv = 0; lv < depth; lv++) {
        const uint32_t v = ks.s[node];
        node = 2 * node + 1 + (sy[v & 0xFFu] >= (v >> 8) ? 1u : 0u);
    }
    const uint32_t size = SUPER_SIZE >> depth, cell = node - ((1u << depth) - 1);
    return sb * SUPER_SIZE + cell * size + size / 2;
}

// NT threads per query: 1024 (one warp per probe search, a single round of 32) when the batch is
// one wave of CTAs, 256 for large batches (more queries resident per SM)
template <int NT>
__global__ void __launch_bounds__(NT) qprep_kernel(const float *__restrict__ queries, uint32_t n,
                                                    const uint4 *__restrict__ skey, const KdSplits *__restrict__ ksplit,
                                                    uint64_t N, uint32_t L,
                                                    uint32_t P, uint32_t Lp, uint32_t *__restrict__ pwin,
                                                    float *__restrict__ qy, double *__restrict__ qpaa,
                                                    uint8_t *__restrict__ qsax, float *__restrict__ lut,
                                                    uint32_t *__restrict__ win, unsigned long long *__restrict__ bsf,
                                                    uint32_t *__restrict__ cand_cnt, uint32_t *__restrict__ near_cnt,
                                                    unsigned long long *__restrict__ near_off, uint32_t *__restrict__ near_cap,
                                                    uint32_t *__restrict__ counters, uint32_t *__restrict__ counters_leaf,
                                                    uint32_t *__restrict__ qmap, Band *__restrict__ qband, float band0,
                                                    uint32_t *__restrict__ bad) {
    __shared__ float row[1024];
    __shared__ double beta[ISAX_NBETA];
    __shared__ double m[W];
    __shared__ uint32_t sym[W];
    __shared__ double stats[2];
    const uint32_t q = blockIdx.x, t = threadIdx.x;
    for (uint32_t i = t; i < n; i += blockDim.x) row[i] = queries[(uint64_t)q * n + i];
    for (uint32_t k = t; k < ISAX_NBETA; k += blockDim.x) beta[k] = c_beta_q[k];
    __syncthreads();
    if (t == 0) {  // C1, strictly left to right (R3): one thread, the same operations as summarise.cu
        double s = 0.0;
        bool finite = true;
        for (uint32_t i = 0; i < n; i++) {
            finite &= isfinite(row[i]);
            s = __dadd_rn(s, (double)row[i]);
        }
        const double mu = __ddiv_rn(s, (double)n);
        double s2 = 0.0;
        for (uint32_t i = 0; i < n; i++) {
            double d = __dsub_rn((double)row[i], mu);
            s2 = __dadd_rn(s2, __dmul_rn(d, d));
        }
        stats[0] = mu;
        stats[1] = __dsqrt_rn(__ddiv_rn(s2, (double)n));
        if (!finite) atomicOr(bad, 1u);
        // reset the per-query state of this batch slot
        cand_cnt[q] = 0;
        near_cnt[q] = 0;
        near_off[q] = (unsigned long long)q * NEAR_K;
        near_cap[q] = NEAR_K;
        counters[4 * q + 0] = counters[4 * q + 1] = counters[4 * q + 2] = counters[4 * q + 3] = 0;
        counters_leaf[q] = 0;
        qmap[q] = q;  // round 0 scans every query of the batch over the band (-1, +inf), all positions (R10)
        qband[q] = Band{-1.0f, band0 > 0.f ? -band0 : __int_as_float(0x7f800000), 0u, (uint32_t)N};
        bsf[q] = ~0ull;
    }
    __syncthreads();
    const double mu = stats[0], sd = stats[1];
    const bool flat = sd < 1e-12;
    for (uint32_t i = t; i < n; i += blockDim.x) {
        const float y = flat ? 0.0f : __double2float_rn(__ddiv_rn(__dsub_rn((double)row[i], mu), sd));
        row[i] = y;
        qy[(uint64_t)q * n + i] = y;
    }
    __syncthreads();
    const uint32_t seg = n / W;
    if (t < W) {  // C2 + C4
        double acc = 0.0;
        for (uint32_t j = 0; j < seg; j++) acc = __dadd_rn(acc, (double)row[t * seg + j]);
        const double mm = __ddiv_rn(acc, (double)seg);
        m[t] = mm;
        sym[t] = sax_symbol(beta, mm);
        qpaa[q * W + t] = mm;
        qsax[q * W + t] = (uint8_t)sym[t];
    }
    __syncthreads();
    // LUT (R7): the fp64 mindist per (segment, symbol), scaled by n/w, rounded down to fp32
    const double segd = (double)seg;
    for (uint32_t e = t; e < W * CARD; e += blockDim.x) {
        const uint32_t s = e >> 8, c = e & 255u;
        const double mm = m[s];
        double d = 0.0;
        if (c > 0 && mm < beta[c - 1]) d = __dsub_rn(beta[c - 1], mm);
        else if (c < CARD - 1 && mm > beta[c]) d = __dsub_rn(mm, beta[c]);
        lut[((uint64_t)q * W + s) * CARD + c] = __double2float_rd(__dmul_rn(segd, __dmul_rn(d, d)));
    }
    // Multi-probe approximate answer (R5). Besides the query's own key, probe the keys obtained
    // by moving the symbols of the P most fragile key bits across their nearest region
    // boundary. The candidates are the plane-0/1 bits whose segment mean lies closest to the
    // breakpoint that flips them. A near-duplicate whose noise flipped an early key bit lands
    // far from its source in the sorted order; one of the probes lands next to it.
    __shared__ uint32_t sel_s[8], sel_c[8];
    if (t < 32 && P > 0) {
        const uint32_t pl = t >> 4, sg = t & 15;
        const uint32_t c = sym[sg], step = 128u >> pl;
        const uint32_t lo_c = (c / step) * step, hi_c = lo_c + step;
        const double mm = m[sg];
        const double dlo = lo_c > 0 ? mm - beta[lo_c - 1] : 1e300;
        const double dhi = hi_c < CARD ? beta[hi_c - 1] - mm : 1e300;
        const uint32_t target = dlo < dhi ? lo_c - 1 : hi_c;
        const float mg = (float)fmin(dlo, dhi);
        uint32_t key = (__float_as_uint(fmaxf(mg, 0.f)) & ~31u) | t;
        for (uint32_t k = 0; k < P; k++) {
            const uint32_t mn = __reduce_min_sync(0xffffffffu, key);
            if (key == mn) {
                sel_s[k] = sg;
                sel_c[k] = target;
                key = 0xffffffffu;
            }
        }
    }
    __syncthreads();
    const uint32_t NP = 1u << P;
    // kd depth of a probe cell: probe_L rows = SUPER_SIZE >> depth (256 -> 2 levels), at most 4
    uint32_t cell_depth = 0, main_depth = 0;
    while (cell_depth < KD_LEVELS && (SUPER_SIZE >> (cell_depth + 1)) >= Lp) cell_depth++;
    while (main_depth < KD_LEVELS && (SUPER_SIZE >> (main_depth + 1)) >= L) main_depth++;
    const uint32_t NX = neighbour_windows(L, P);  // 2 extra windows (see neighbour_windows)
    const uint32_t warp = t >> 5, lane = t & 31;
    for (uint32_t j = warp; j < NP; j += blockDim.x / 32) {  // locate each probe key, one warp per probe
        uint32_t sy[W];
#pragma unroll
        for (int s2 = 0; s2 < W; s2++) sy[s2] = sym[s2];
        for (uint32_t b = 0; b < P; b++)
            if ((j >> b) & 1u) sy[sel_s[b]] = sel_c[b];
        const uint4 kq = isax_key(sy);
        // super-node of the key (R5, R6b): the last one whose smallest key is below it
        const uint64_t nsup = (N + SUPER_SIZE - 1) / SUPER_SIZE;
        uint64_t lo = 0, hi = nsup;
        while (hi - lo > 32) {
            const uint64_t span = hi - lo;
            const uint64_t p = lo + (span * (lane + 1)) / 33;
            const bool less = key_less(__ldg(skey + p), kq);
            const uint32_t bal = __ballot_sync(0xffffffffu, less);
            const uint32_t c = __popc(bal);  // probes are increasing, so `less` is a prefix
            const uint64_t p_last = __shfl_sync(0xffffffffu, p, (c == 0 ? 0 : c - 1));
            const uint64_t p_next = __shfl_sync(0xffffffffu, p, (c == 32 ? 31 : c));
            if (c == 0) hi = p_next;
            else {
                lo = p_last + 1;
                if (c < 32) hi = p_next;
            }
        }
        const bool less = (lo + lane < hi) && key_less(__ldg(skey + lo + lane), kq);
        const uint64_t c = lo + __popc(__ballot_sync(0xffffffffu, less));
        const uint64_t sq = c > 0 ? c - 1 : 0;
        if (lane == 0) {
            const uint32_t len = j == 0 ? L : Lp;
            // the main window is whole super-nodes around that one: with an odd count (L = 1024,
            // 3072) it is centred on it, with an even count (2048) it is it and the next. The keys
            // just below the query's are at its end or in the one before, the keys just above in
            // it or the next. A probe window sits on the kd cell of its super-node (probe_L rows)
            // that the first kd splits send the probe's symbols to.
            uint64_t pos = sq * SUPER_SIZE + SUPER_SIZE / 2 + (((L / SUPER_SIZE) & 1u) ? 0u : SUPER_SIZE / 2);
            if (j > 0) pos = kd_cell_centre(ksplit, sq, sy, cell_depth);
            else if (L < SUPER_SIZE) pos = kd_cell_centre(ksplit, sq, sy, main_depth);  // a cell of the super-node
            uint64_t start = 0;
            if (N > len) {
                const int64_t s0 = (int64_t)pos - (int64_t)(len / 2);
                const int64_t smax = (int64_t)(N - len);
                start = (uint64_t)(s0 < 0 ? 0 : (s0 > smax ? smax : s0));
            }
            if (j == 0) {
                win[2 * q] = (uint32_t)start;
                win[2 * q + 1] = (uint32_t)(start + (N > len ? len : N));
                if (NX) {  // the kd-descended quarters of the neighbouring super-nodes (R5, R6b)
                    for (uint32_t k = 0; k < 2; k++) {
                        uint64_t sn = k == 0 ? (sq > 0 ? sq - 1 : sq + 1) : (sq + 1 < nsup ? sq + 1 : (sq > 0 ? sq - 1 : sq));
                        sn = sn < nsup ? sn : nsup - 1;
                        const uint64_t p2 = kd_cell_centre(ksplit, sn, sy, cell_depth);
                        uint64_t st2 = 0;
                        if (N > Lp) {
                            const int64_t a = (int64_t)p2 - (int64_t)(Lp / 2), smax = (int64_t)(N - Lp);
                            st2 = (uint64_t)(a < 0 ? 0 : (a > smax ? smax : a));
                        }
                        pwin[q * MAX_PROBES + NP - 1 + k] = (uint32_t)st2;
                    }
                }
            } else {
                pwin[q * MAX_PROBES + j - 1] = (uint32_t)start;
            }
        }
    }
    __syncthreads();
    // keep the probe windows that add rows: drop those inside the main window (already refined)
    // and repeats of an earlier start; their count goes into the last slot. Warp 0, lane = probe.
    if (warp == 0) {
        uint32_t *pw = pwin + (uint64_t)q * MAX_PROBES;
        const uint32_t np = NP - 1 + NX, lp = (uint32_t)(N < Lp ? N : Lp);
        const uint32_t ws = win[2 * q], we = win[2 * q + 1];
        const uint32_t a = lane < np ? pw[lane] : 0xFFFFFFFFu;
        const bool rep = (__match_any_sync(0xffffffffu, a) & ((1u << lane) - 1u)) != 0;
        const bool keep = lane < np && !rep && !(a >= ws && a + lp <= we);
        const uint32_t kb = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) pw[__popc(kb & ((1u << lane) - 1u))] = a;
        if (lane == 0) pw[MAX_PROBES - 1] = __popc(kb);
    }
}

void launch_qprep(const isax_index *ix, const float *queries, uint32_t Q, float band0, cudaStream_t s, uint32_t *bad) {
    const QueryScratch &qs = ix->qs;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    auto kern = Q <= (uint32_t)(2 * sms) ? qprep_kernel<1024> : qprep_kernel<256>;
    kern<<<Q, Q <= (uint32_t)(2 * sms) ? 1024 : 256, 0, s>>>(queries, ix->n, ix->skey, ix->ksplit, ix->N,
                                   ix->win_L, probe_bits(ix), ix->pr_L, qs.pwin, qs.qy, qs.qpaa, qs.qsax, qs.lut, qs.win, qs.bsf, qs.cand_cnt,
                                   qs.near_cnt, qs.near_off, qs.near_cap, qs.counters, qs.counters_leaf, qs.qmap, qs.qband,
                                   band0, bad);
}

// ------------------------------------------------------------------------------------ window
// d^2 of one row by one warp: lane holds elements [k*128 + 4*lane, +4) for k < NS.
template <int NS>
__device__ __forceinline__ float row_d2(const float *__restrict__ row, const float4 (&qv)[NS], uint32_t n,
                                        uint32_t lane) {
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < NS; k++) {
        const uint32_t i = k * 128 + 4 * lane;
        if (i < n) {
            const float4 v = __ldcs(reinterpret_cast<const float4 *>(row + i));
            float d;
            d = v.x - qv[k].x; acc = fmaf(d, d, acc);
            d = v.y - qv[k].y; acc = fmaf(d, d, acc);
            d = v.z - qv[k].z; acc = fmaf(d, d, acc);
            d = v.w - qv[k].w; acc = fmaf(d, d, acc);
        }
    }
    return warp_sum(acc);
}

// The rows of one query (main window, then probe windows) are split over several CTAs of
// WIN_ROWS rows each, so a batch keeps every SM busy (256: finer than 512 against the uneven last
// wave, 0.092 -> 0.079 ms at cfg3; 128 lengthens the near lists). Each warp refines four rows at a
// time, with all their loads in flight. Each CTA folds its minimum into the global packed BSF. It then appends
// the rows within (1 + delta) of the BSF it reads back. That BSF can only be >= the final one, so
// the near list is a superset of the final near ties (R9).
#ifndef ISAX_WIN_ROWS
#define ISAX_WIN_ROWS 256
#endif
constexpr uint32_t WIN_ROWS = ISAX_WIN_ROWS;

template <int NS>
__global__ void __launch_bounds__(256) window_kernel(const float *__restrict__ stored, const uint32_t *__restrict__ perm,
                                                     uint32_t n, uint64_t N, const float *__restrict__ qy,
                                                     const uint32_t *__restrict__ win, const uint32_t *__restrict__ pwin,
                                                     uint32_t nprobe, uint32_t Lp, const uint32_t *__restrict__ qmap,
                                                     unsigned long long *__restrict__ bsf, NearList nl,
                                                     uint32_t *__restrict__ counters, float onepd) {
    __shared__ float d2s[WIN_ROWS];
    __shared__ unsigned long long smin;
    __shared__ unsigned long long cur;
    const uint32_t q = qmap ? qmap[blockIdx.y] : blockIdx.y;
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t ws = win[2 * q], we = win[2 * q + 1], L = we - ws;
    const uint32_t lp = (uint32_t)(N < Lp ? N : Lp);
    const uint32_t rows = L + (nprobe ? pwin[q * MAX_PROBES + MAX_PROBES - 1] : 0u) * lp;  // kept probes (qprep)
    const uint32_t r0 = blockIdx.x * WIN_ROWS;
    if (r0 >= rows) return;
    const uint32_t r1 = min(rows, r0 + WIN_ROWS);
    ISAX_BOUND(ws <= we && we <= N);
    auto row_pos = [&](uint32_t r) -> uint32_t {
        if (r < L) return ws + r;
        r -= L;
        const uint32_t p = pwin[q * MAX_PROBES + r / lp] + r % lp;
        ISAX_BOUND(r / lp < MAX_PROBES - 1 && p < N);
        return p;
    };
    float4 qv[NS];
#pragma unroll
    for (int k = 0; k < NS; k++) {
        const uint32_t i = k * 128 + 4 * lane;
        qv[k] = i < n ? *reinterpret_cast<const float4 *>(qy + (uint64_t)q * n + i) : make_float4(0, 0, 0, 0);
    }
    if (t == 0) smin = ~0ull;
    __syncthreads();
    // four rows per warp step, all their loads in flight before any reduction; the warp's minimum
    // is tracked as (d^2 bits, row) and its id is looked up once at the end (the answer itself
    // comes from the near list, R9; the id in the BSF word is only a fallback)
    constexpr int RW = 4;
    unsigned long long mine = ~0ull;
    for (uint32_t r = r0 + warp * RW; r < r1; r += 8 * RW) {
        const float *rp[RW];
#pragma unroll
        for (int j = 0; j < RW; j++) rp[j] = stored + (uint64_t)row_pos(r + j < r1 ? r + j : r) * n;
        float4 v[RW][NS];
#pragma unroll
        for (int k = 0; k < NS; k++) {
            const uint32_t i = k * 128 + 4 * lane;
#pragma unroll
            for (int j = 0; j < RW; j++)
                v[j][k] = i < n ? __ldcs(reinterpret_cast<const float4 *>(rp[j] + i)) : make_float4(0, 0, 0, 0);
        }
        float a[RW];
#pragma unroll
        for (int j = 0; j < RW; j++) {
            float s = 0.f;
#pragma unroll
            for (int k = 0; k < NS; k++) {
                if (k * 128 + 4 * lane < n) {
                    float d;
                    d = v[j][k].x - qv[k].x; s = fmaf(d, d, s);
                    d = v[j][k].y - qv[k].y; s = fmaf(d, d, s);
                    d = v[j][k].z - qv[k].z; s = fmaf(d, d, s);
                    d = v[j][k].w - qv[k].w; s = fmaf(d, d, s);
                }
            }
            a[j] = warp_sum(s);
        }
        if (lane == 0) {
#pragma unroll
            for (int j = 0; j < RW; j++) {
                if (r + j < r1) {
                    d2s[r + j - r0] = a[j];
                    const unsigned long long p = pack_bsf(a[j], r + j);
                    mine = p < mine ? p : mine;
                }
            }
        }
    }
    if (lane == 0 && mine != ~0ull) mine = pack_bsf(bsf_d2(mine), perm[row_pos((uint32_t)mine)]);
    if (lane == 0) atomicMin(&smin, mine);
    __syncthreads();
    if (t == 0) {
        atomicMin(&bsf[q], smin);
        cur = atomicAdd(&bsf[q], 0ull);
        atomicAdd(&counters[4 * q + 3], r1 - r0);  // window rows (stats; "refined" counts candidates only)
    }
    __syncthreads();
    const float lim = bsf_d2(cur) * onepd;
    for (uint32_t r = r0 + t; r < r1; r += blockDim.x) {
        if (d2s[r - r0] <= lim) {
            const uint32_t pos = row_pos(r);
            near_append(nl, q, perm[pos], pos, d2s[r - r0]);
        }
    }
}

uint32_t probe_bits(const isax_index *ix) {
    return ix->opts.probe_bits == ISAX_PROBES_NONE ? 0u : ix->opts.probe_bits;
}

uint32_t window_probes(const isax_index *ix) {
    return (1u << probe_bits(ix)) - 1 + neighbour_windows(ix->win_L, probe_bits(ix));
}

void launch_window(const isax_index *ix, uint32_t Q, const uint32_t *qmap, float delta, cudaStream_t s) {
    const QueryScratch &qs = ix->qs;
    const float onepd = 1.0f + delta;
    const uint32_t ns = (ix->n + 127) / 128;
    const uint32_t nprobe = (1u << probe_bits(ix)) - 1 + neighbour_windows(ix->win_L, probe_bits(ix));
    const uint32_t lp = (uint32_t)(ix->N < ix->pr_L ? ix->N : ix->pr_L);
    const uint32_t L = (uint32_t)(ix->N < ix->win_L ? ix->N : ix->win_L);
    const uint32_t rows = L + nprobe * lp;
    const dim3 grid((rows + WIN_ROWS - 1) / WIN_ROWS, Q);
#define WIN_CASE(K)                                                                                          \
    case K:                                                                                                  \
        window_kernel<K><<<grid, 256, 0, s>>>(ix->stored, ix->perm, ix->n, ix->N, qs.qy, qs.win, qs.pwin,    \
                                              nprobe, ix->pr_L, qmap, qs.bsf,                         \
                                              NearList{qs.near, qs.near_off, qs.near_cap, qs.near_cnt},       \
                                              qs.counters, onepd);                                           \
        break;
    switch (ns) {
        WIN_CASE(1) WIN_CASE(2) WIN_CASE(3) WIN_CASE(4) WIN_CASE(5) WIN_CASE(6) WIN_CASE(7) WIN_CASE(8)
    }
#undef WIN_CASE
}

// ------------------------------------------------------------------------------------ LB dump
// Debug / parity: LB^2 of a range of sorted positions, accumulated exactly as lbscan does it
// (fp32, segments 0..15 left to right).
__global__ void lb_dump_kernel(const uint4 *__restrict__ sax, const float *__restrict__ lut, uint32_t Q,
                               uint64_t first, uint64_t count, float *__restrict__ out) {
    const uint32_t q = blockIdx.y;
    const float *L = lut + (uint64_t)q * W * CARD;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 wv = sax[first + i];
        const uint32_t v[4] = {wv.x, wv.y, wv.z, wv.w};
        float lb = 0.f;
#pragma unroll
        for (int s = 0; s < W; s++) lb += L[s * CARD + ((v[s >> 2] >> (8 * (s & 3))) & 0xFFu)];
        out[(uint64_t)q * count + i] = lb;
    }
}

void launch_lb_dump(const isax_index *ix, uint32_t Q, uint64_t first_pos, uint64_t count, float *out,
                    cudaStream_t s) {
    if (!count || !Q) return;
    const dim3 grid((unsigned)umin64((count + 255) / 256, 1184), Q);
    lb_dump_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const uint4 *>(ix->sax), ix->qs.lut, Q, first_pos, count,
                                        out);
}

}  // namespace isax
