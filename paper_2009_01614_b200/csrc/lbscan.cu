// lbscan.cu: the lower-bound scan over every iSAX summary, with candidate compaction.
//
// "a number of lower bound calculation workers compute the lower bound distances
// between the query and the iSAX summary of each data series ... and prune the series whose
// lower bound distance is larger than the approximate real distance computed earlier. The data
// series that are not pruned, are stored in a candidate list". north_star (b): "a full scan of
// mindist_PAA_iSAX lower bounds over all summaries, compaction of the unpruned candidates".
//
// v1 design:
//  - Each CTA serves a group of G queries. Their fp32 LUTs (16 x 256 x 4 B = 16 KB each) sit
//    in shared memory, so one pass over the SAX array serves G queries: HBM traffic is
//    16 B x N per G queries.
//  - Each thread streams 16-byte words with ld.global.nc.L1::no_allocate (no reuse), U words
//    in flight per thread.
//  - LB^2 = sum over segments 0..15, left to right in fp32 (the same order as
//    isax_query_debug). A position is kept iff LB^2 <= T = bsf^2 * (1 + delta) and it lies
//    outside the window (R8).
//  - Compaction: __ballot_sync, then one atomicAdd per warp per query with survivors, then
//    each kept lane writes its position at base + popc(ballot & lanemask_lt).
#include "isax_device.cuh"

namespace isax {

__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

constexpr int LB_THREADS = 256;
constexpr int LB_U = 4;

template <int G>
__global__ void __launch_bounds__(LB_THREADS) lbscan_kernel(const uint4 *__restrict__ sax, uint32_t N,
                                                            const float *__restrict__ lut_all,
                                                            const uint32_t *__restrict__ qmap,
                                                            const uint32_t *__restrict__ qrange, uint32_t nq,
                                                            uint32_t scan_lo, uint32_t scan_hi,
                                                            const unsigned long long *__restrict__ bsf,
                                                            const uint32_t *__restrict__ win, float onepd,
                                                            uint32_t *__restrict__ cand,
                                                            uint32_t *__restrict__ cand_cnt, uint32_t cap) {
    extern __shared__ __align__(16) float slut[];  // [G][16][256]
    __shared__ float T[G];
    __shared__ uint32_t ws[G], we[G], r0[G], r1[G], qid[G];
    const uint32_t t = threadIdx.x, lane = t & 31;
    const uint32_t g0 = blockIdx.y * G;
    for (uint32_t e = t; e < G * W * CARD; e += LB_THREADS) {
        const uint32_t g = e / (W * CARD);
        const uint32_t qi = g0 + g < nq ? qmap[g0 + g] : qmap[g0];
        slut[e] = lut_all[(uint64_t)qi * W * CARD + (e % (W * CARD))];
    }
    if (t < G) {
        const bool valid = g0 + t < nq;
        const uint32_t qi = valid ? qmap[g0 + t] : 0;
        qid[t] = qi;
        T[t] = valid ? bsf_d2(bsf[qi]) * onepd : -1.0f;  // an invalid slot keeps nothing
        ws[t] = win[2 * qi];
        we[t] = win[2 * qi + 1];
        r0[t] = valid ? qrange[2 * (g0 + t)] : 0;
        r1[t] = valid ? qrange[2 * (g0 + t) + 1] : 0;
    }
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
    const uint64_t step = (uint64_t)gridDim.x * LB_THREADS * LB_U;
    for (uint64_t base = scan_lo + (uint64_t)blockIdx.x * LB_THREADS * LB_U; base < scan_hi; base += step) {
        uint4 wv[LB_U];
#pragma unroll
        for (int u = 0; u < LB_U; u++) {
            const uint64_t pos = base + u * LB_THREADS + t;
            wv[u] = pos < scan_hi ? ld_stream(sax + pos) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < LB_U; u++) {
            const uint32_t pos = (uint32_t)(base + u * LB_THREADS + t);
            const bool inr = base + u * LB_THREADS + t < scan_hi;
            const uint32_t v[4] = {wv[u].x, wv[u].y, wv[u].z, wv[u].w};
#pragma unroll
            for (int g = 0; g < G; g++) {
                const float *L = slut + g * W * CARD;
                float lb = 0.f;
#pragma unroll
                for (int s = 0; s < W; s++) lb += L[s * CARD + ((v[s >> 2] >> (8 * (s & 3))) & 0xFFu)];
                const bool keep = inr && lb <= T[g] && (pos < ws[g] || pos >= we[g]) && pos >= r0[g] && pos < r1[g];
                const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                if (bal) {
                    uint32_t off = 0;
                    if (lane == 0) off = atomicAdd(&cand_cnt[qid[g]], (uint32_t)__popc(bal));
                    off = __shfl_sync(0xffffffffu, off, 0);
                    if (keep) {
                        const uint32_t k = off + __popc(bal & lt);
                        if (k < cap) cand[(uint64_t)qid[g] * cap + k] = pos;
                    }
                }
            }
        }
    }
}

template <int G>
static void launch_g(const isax_index *ix, uint32_t nq, const uint32_t *qmap, const uint32_t *qrange, uint32_t lo,
                     uint32_t hi, float onepd, cudaStream_t s) {
    const size_t smem = (size_t)G * W * CARD * sizeof(float);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(lbscan_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t groups = (nq + G - 1) / G;
    const int per_sm = std::max(1, (int)((227 * 1024) / (smem + 2048)));
    const uint64_t tiles = ((uint64_t)(hi - lo) + LB_THREADS * LB_U - 1) / (LB_THREADS * LB_U);
    uint64_t gx = ((uint64_t)sms * per_sm + groups - 1) / groups;
    gx = std::max<uint64_t>(1, umin64(gx, tiles));
    const dim3 grid((unsigned)gx, groups);
    const QueryScratch &qs = ix->qs;
    lbscan_kernel<G><<<grid, LB_THREADS, smem, s>>>(reinterpret_cast<const uint4 *>(ix->sax), (uint32_t)ix->N, qs.lut,
                                                   qmap, qrange, nq, lo, hi, qs.bsf, qs.win, onepd, qs.cand,
                                                   qs.cand_cnt, qs.cand_cap);
}

// ------------------------------------------------------------------------------------ leaf scan
// v2, the default: the MESSI idea on the sorted array. P:346-349: "the index workers traverse
// the index subtrees ... using BSF to decide which subtrees will be pruned"; leaves that
// survive are examined "by first computing lower bound distances using the iSAX summaries".
//
// A leaf is LEAF consecutive sorted positions. Its node summary (build: leaf_meta_kernel) is the
// per-segment [min, max] symbol. The node's region on segment s is [beta_min, beta_{max+1}), and
// its MINDIST term is min over c in [min, max] of LUT[s][c]. LUT[s][.] is V-shaped around the
// query's own symbol q_s (zero there, growing away from it), so that minimum is
// LUT[s][clamp(q_s, min, max)]: one lookup per segment per leaf.
//   node LB^2 <= LB^2 of every member (termwise <=, and fp32 addition is monotone)
// A leaf is pruned iff node LB^2 > T (1 + 2^-19). The extra 2^-19 covers the different fp32
// summation order of the warp reduction (16 terms: < 2^-20 relative). Members of surviving
// leaves get the exact per-series test of v1, so the candidate set is exactly v1's.
//
// Work unit: one warp, two leaves. Lane = (leaf half, segment). The node LB needs 1 lookup +
// 4 xor-shuffle adds per leaf per query. A leaf's 64 words (1 KB) are read only if some query
// of the CTA's group keeps it.
constexpr uint32_t LEAF = 64;

constexpr int LF_THREADS = 1024;  // one CTA per SM; all 32 warps share the group's LUTs

template <int G>
__global__ void __launch_bounds__(LF_THREADS, 1) leafscan_kernel(
    const uint4 *__restrict__ sax, const uint8_t *__restrict__ lmeta, uint32_t N, const float *__restrict__ lut_all,
    const uint8_t *__restrict__ qsax_all, const uint32_t *__restrict__ qmap, const uint32_t *__restrict__ qrange,
    uint32_t nq, uint32_t leaf_lo, uint32_t leaf_hi, const unsigned long long *__restrict__ bsf,
    const uint32_t *__restrict__ win, float onepd, uint32_t *__restrict__ cand, uint32_t *__restrict__ cand_cnt,
    uint32_t cap, uint32_t *__restrict__ leaves_alive, unsigned long long *__restrict__ leaf_loads) {
    extern __shared__ __align__(16) float slut[];  // [G][16][256]
    __shared__ float T[G], Tb[G];
    __shared__ uint32_t ws[G], we[G], r0[G], r1[G], qid[G];
    __shared__ uint8_t qs[G][W];
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t g0 = blockIdx.y * G;
    for (uint32_t e = t; e < G * W * CARD; e += LF_THREADS) {
        const uint32_t g = e / (W * CARD);
        const uint32_t qi = g0 + g < nq ? qmap[g0 + g] : qmap[g0];
        slut[e] = lut_all[(uint64_t)qi * W * CARD + (e % (W * CARD))];
    }
    if (t < G * W) {
        const uint32_t g = t / W;
        const uint32_t qi = g0 + g < nq ? qmap[g0 + g] : qmap[g0];
        qs[g][t % W] = qsax_all[qi * W + t % W];
    }
    if (t < G) {
        const bool valid = g0 + t < nq;
        const uint32_t qi = valid ? qmap[g0 + t] : 0;
        qid[t] = qi;
        const float tq = valid ? bsf_d2(bsf[qi]) * onepd : -1.0f;
        T[t] = tq;
        Tb[t] = tq * (1.0f + 0x1.0p-19f);
        ws[t] = win[2 * qi];
        we[t] = win[2 * qi + 1];
        r0[t] = valid ? qrange[2 * (g0 + t)] : 0;
        r1[t] = valid ? qrange[2 * (g0 + t) + 1] : 0;
    }
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t seg = lane & 15, half = lane >> 4;
    const uint32_t wstride = gridDim.x * (LF_THREADS / 32) * 2;
    uint32_t alive_cnt = 0;  // lane g counts the leaves that survived for query g
    uint32_t loads = 0;      // lane 0 counts the leaves whose words were read
    uint32_t lp = leaf_lo + (blockIdx.x * (LF_THREADS / 32) + warp) * 2;
    // software pipeline: the node summary of the next leaf pair is in flight while this one is used
    uint32_t mn_n = 0, mx_n = 255;
    if (lp + half < leaf_hi) {
        mn_n = __ldg(lmeta + (uint64_t)(lp + half) * 32 + seg);
        mx_n = __ldg(lmeta + (uint64_t)(lp + half) * 32 + 16 + seg);
    }
    for (; lp < leaf_hi; lp += wstride) {
        const uint32_t leaf = lp + half;
        const bool lval = leaf < leaf_hi;
        const uint32_t mn = mn_n, mx = mx_n;
        const uint32_t nxt = lp + wstride + half;
        if (nxt < leaf_hi) {
            mn_n = __ldg(lmeta + (uint64_t)nxt * 32 + seg);
            mx_n = __ldg(lmeta + (uint64_t)nxt * 32 + 16 + seg);
        }
        const uint32_t p0 = leaf * LEAF, p1 = min(p0 + LEAF, N);
        uint32_t alive = 0;
#pragma unroll
        for (int g = 0; g < G; g++) {
            const uint32_t c = min(max((uint32_t)qs[g][seg], mn), mx);
            float v = slut[g * W * CARD + seg * CARD + c];
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            // the leaf must hold a position of this slot's range that is outside the window
            const bool in_range = p0 < r1[g] && p1 > r0[g];
            const bool all_win = p0 >= ws[g] && p1 <= we[g];
            if (lval && v <= Tb[g] && in_range && !all_win) alive |= 1u << g;
        }
#pragma unroll 1
        for (int h = 0; h < 2; h++) {
            const uint32_t am = __shfl_sync(0xffffffffu, alive, h * 16);
            if (!am) continue;
            loads++;
            alive_cnt += (am >> lane) & 1u;
            const uint32_t base = (lp + h) * LEAF;
            uint4 wv[2];
#pragma unroll
            for (int u = 0; u < 2; u++) {
                const uint32_t pos = base + u * 32 + lane;
                wv[u] = pos < N ? ld_stream(sax + pos) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int g = 0; g < G; g++) {
                if (!((am >> g) & 1u)) continue;
                const float *L = slut + g * W * CARD;
#pragma unroll
                for (int u = 0; u < 2; u++) {
                    const uint32_t pos = base + u * 32 + lane;
                    const uint32_t v[4] = {wv[u].x, wv[u].y, wv[u].z, wv[u].w};
                    float lb = 0.f;
#pragma unroll
                    for (int s = 0; s < W; s++) lb += L[s * CARD + ((v[s >> 2] >> (8 * (s & 3))) & 0xFFu)];
                    const bool keep = pos < N && lb <= T[g] && (pos < ws[g] || pos >= we[g]) && pos >= r0[g] &&
                                      pos < r1[g];
                    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                    if (bal) {
                        uint32_t off = 0;
                        if (lane == 0) off = atomicAdd(&cand_cnt[qid[g]], (uint32_t)__popc(bal));
                        off = __shfl_sync(0xffffffffu, off, 0);
                        if (keep) {
                            const uint32_t k = off + __popc(bal & lt);
                            if (k < cap) cand[(uint64_t)qid[g] * cap + k] = pos;
                        }
                    }
                }
            }
        }
    }
    if (lane < G && alive_cnt && g0 + lane < nq) atomicAdd(&leaves_alive[qid[lane]], alive_cnt);
    if (lane == 0 && loads) atomicAdd(leaf_loads, (unsigned long long)loads);
}

template <int G>
static void launch_leaf(const isax_index *ix, uint32_t nq, const uint32_t *qmap, const uint32_t *qrange, uint32_t lo,
                        uint32_t hi, float onepd, cudaStream_t s) {
    const size_t smem = (size_t)G * W * CARD * sizeof(float);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(leafscan_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t groups = (nq + G - 1) / G;
    const uint32_t leaf_lo = lo / LEAF, leaf_hi = (hi + LEAF - 1) / LEAF;
    const uint64_t units = ((uint64_t)(leaf_hi - leaf_lo) + 2 * (LF_THREADS / 32) - 1) / (2 * (LF_THREADS / 32));
    uint64_t gx = ((uint64_t)sms * 4 + groups - 1) / groups;  // ~4 waves of one CTA per SM
    gx = std::max<uint64_t>(1, umin64(gx, units));
    const dim3 grid((unsigned)gx, groups);
    const QueryScratch &qs = ix->qs;
    leafscan_kernel<G><<<grid, LF_THREADS, smem, s>>>(
        reinterpret_cast<const uint4 *>(ix->sax), ix->lmeta, (uint32_t)ix->N, qs.lut, qs.qsax, qmap, qrange, nq,
        leaf_lo, leaf_hi, qs.bsf, qs.win, onepd, qs.cand, qs.cand_cnt, qs.cand_cap, qs.counters_leaf,
        qs.leaf_loads);
}

uint64_t launch_lbscan(const isax_index *ix, uint32_t nq, const uint32_t *qmap, const uint32_t *qrange, uint32_t lo,
                       uint32_t hi, float delta, cudaStream_t s) {
    if (!nq || hi <= lo) return 0;
    const float onepd = 1.0f + delta;
    if (ix->opts.flags & ISAX_FLAG_FLAT_SCAN) {  // ParIS flat scan (v1), kept for A/B measurement
        const uint32_t G = nq >= 4 ? 4 : nq;
        if (G == 4) launch_g<4>(ix, nq, qmap, qrange, lo, hi, onepd, s);
        else if (G == 3) launch_g<3>(ix, nq, qmap, qrange, lo, hi, onepd, s);
        else if (G == 2) launch_g<2>(ix, nq, qmap, qrange, lo, hi, onepd, s);
        else launch_g<1>(ix, nq, qmap, qrange, lo, hi, onepd, s);
        return 16ull * (hi - lo) * ((nq + G - 1) / G);  // words read
    }
    const uint32_t G = nq >= 8 ? 8 : nq >= 4 ? 4 : nq >= 2 ? 2 : 1;
    if (G == 8) launch_leaf<8>(ix, nq, qmap, qrange, lo, hi, onepd, s);
    else if (G == 4) launch_leaf<4>(ix, nq, qmap, qrange, lo, hi, onepd, s);
    else if (G == 2) launch_leaf<2>(ix, nq, qmap, qrange, lo, hi, onepd, s);
    else launch_leaf<1>(ix, nq, qmap, qrange, lo, hi, onepd, s);
    const uint64_t leaves = (hi + LEAF - 1) / LEAF - lo / LEAF;
    return 32ull * leaves * ((nq + G - 1) / G);  // node summaries read; leaf words are counted on the device
}

// ------------------------------------------------------------------------------------ leaf meta
// Build: per leaf, the per-segment min and max symbol of its (up to) LEAF members, 32 bytes.
__global__ void leaf_meta_kernel(const uint4 *__restrict__ sax, uint64_t N, uint8_t *__restrict__ lmeta) {
    const uint64_t nleaf = (N + LEAF - 1) / LEAF;
    for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < nleaf; l += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t mn[4] = {~0u, ~0u, ~0u, ~0u}, mx[4] = {0, 0, 0, 0};
        const uint64_t p1 = umin64(N, (l + 1) * LEAF);
        for (uint64_t p = l * LEAF; p < p1; p++) {
            const uint4 w = __ldg(sax + p);
            const uint32_t v[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int k = 0; k < 4; k++) {
                mn[k] = __vminu4(mn[k], v[k]);
                mx[k] = __vmaxu4(mx[k], v[k]);
            }
        }
        uint4 *o = reinterpret_cast<uint4 *>(lmeta + l * 32);
        o[0] = make_uint4(mn[0], mn[1], mn[2], mn[3]);
        o[1] = make_uint4(mx[0], mx[1], mx[2], mx[3]);
    }
}

void launch_leaf_meta(const uint8_t *sax, uint64_t N, uint8_t *lmeta, cudaStream_t s) {
    const uint64_t nleaf = (N + LEAF - 1) / LEAF;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, umin64((nleaf + 255) / 256, 148 * 16));
    leaf_meta_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const uint4 *>(sax), N, lmeta);
}

}  // namespace isax
