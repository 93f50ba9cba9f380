// lbscan.cu: the lower-bound scan over every iSAX summary, with candidate compaction.
//
// "a number of lower bound calculation workers compute the lower bound distances
// between the query and the iSAX summary of each data series ... and prune the series whose
// lower bound distance is larger than the approximate real distance computed earlier. The data
// series that are not pruned, are stored in a candidate list". north_star (b): "a full scan of
// mindist_PAA_iSAX lower bounds over all summaries, compaction of the unpruned candidates".
//
// Keep rule, per query slot (R8, R10): a position p outside the window is a candidate iff
//     band_lo < LB^2(p) <= T,   T = min(band_hi, bsf^2 (1 + delta))
// LB^2 is the fp32 sum of LUT[s][sym_s] over s = 0..15, left to right, the same order as
// isax_query_debug. Round 0 uses band (-1, +inf). When a query's list overflows, the host
// shrinks band_hi with the per-query LB histogram, so the smallest bounds are refined first
// (MESSI's priority-queue order, done in LB bands). The next band then starts
// where the previous one ended.
//
// The scans:
//  - nodescan_kernel + itemscan_kernel (default): MESSI-style node pruning on the sorted array over
//    four node levels (R11, R11c): hyper-node, super-node | leaf, 8-row kd cell, member.
//  - lbscan_kernel (ISAX_FLAG_FLAT_SCAN): the ParIS flat scan of every 16-byte word (A/B).
//  - leafscan_kernel (-DISAX_SCAN_V1=1): the round-2b single-kernel node scan over three levels (A/B).
#include "isax_device.cuh"

namespace isax {

__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ uint32_t byte_of(const uint32_t (&v)[4], int s) { return (v[s >> 2] >> (8 * (s & 3))) & 0xFFu; }

// packed 16-bit lane min / max (native on sm_90+; the byte-lane __vminu4 is emulated)
__device__ __forceinline__ uint32_t max_u16x2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t min_u16x2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
// bytes (b0, b1, b2, b3) of w -> u16x2 (b0, b1) and (b2, b3)
__device__ __forceinline__ uint32_t lo_u16x2(uint32_t w) { return __byte_perm(w, 0u, 0x4140); }
__device__ __forceinline__ uint32_t hi_u16x2(uint32_t w) { return __byte_perm(w, 0u, 0x4342); }

// the fp32 LB^2 of one word against one LUT, segments 0..15 left to right
__device__ __forceinline__ float word_lb(const float *L, const uint4 &wv) {
    const uint32_t v[4] = {wv.x, wv.y, wv.z, wv.w};
    float lb = 0.f;
#pragma unroll
    for (int s = 0; s < W; s++) lb += L[s * CARD + byte_of(v, s)];
    return lb;
}

// sum of the u8 LUT entries of one word. ub is the shared address of the query's [16][256] u8
// table (256-aligned, < 2^24): PRMT merges symbol byte s into the low byte of ub, and the segment
// offset s * 256 becomes the load's immediate.
__device__ __forceinline__ uint32_t ld_sh_u8(uint32_t addr) {
    uint32_t r;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(r) : "r"(addr));
    return r;
}
__device__ __forceinline__ uint32_t word_e8(uint32_t ub, const uint4 &wv, uint32_t &hi) {
    const uint32_t v[4] = {wv.x, wv.y, wv.z, wv.w};
    uint32_t lo = 0;
    hi = 0;
#pragma unroll
    for (int s = 0; s < W / 2; s++) lo += ld_sh_u8(__byte_perm(v[s >> 2], ub, 0x7650u | (uint32_t)(s & 3)) + s * CARD);
#pragma unroll
    for (int s = W / 2; s < W; s++) hi += ld_sh_u8(__byte_perm(v[s >> 2], ub, 0x7650u | (uint32_t)(s & 3)) + s * CARD);
    return lo + hi;  // (hi: the u8 bound of the second half's segments 8..15, R16)
}
// u8 node bound (R11, R11b) of a node summary (per-segment min mn, max mx) against one query:
// q holds the query's symbols as 8 u16x2 pairs; each term is the table entry at the clamped
// symbol, clamp(q_s, mn_s, mx_s), done two segments at a time with u16x2 min / max.
__device__ __forceinline__ uint32_t node_e8(uint32_t ub, const uint4 &qa, const uint4 &qb, const uint4 &mn4,
                                           const uint4 &mx4) {
    const uint32_t qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
    const uint32_t mn[8] = {lo_u16x2(mn4.x), hi_u16x2(mn4.x), lo_u16x2(mn4.y), hi_u16x2(mn4.y),
                            lo_u16x2(mn4.z), hi_u16x2(mn4.z), lo_u16x2(mn4.w), hi_u16x2(mn4.w)};
    const uint32_t mx[8] = {lo_u16x2(mx4.x), hi_u16x2(mx4.x), lo_u16x2(mx4.y), hi_u16x2(mx4.y),
                            lo_u16x2(mx4.z), hi_u16x2(mx4.z), lo_u16x2(mx4.w), hi_u16x2(mx4.w)};
    uint32_t es = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const uint32_t c2 = min_u16x2(max_u16x2(qv[k], mn[k]), mx[k]);
        es += ld_sh_u8(__byte_perm(c2, ub, 0x7650u) + (2 * k) * CARD);
        es += ld_sh_u8(__byte_perm(c2, ub, 0x7652u) + (2 * k + 1) * CARD);
    }
    return es;
}

// node_e8 on summaries already unpacked to u16x2 pairs (unpack_u16x2): for a caller that tests one
// summary against several queries
__device__ __forceinline__ void unpack_u16x2(const uint4 &v, uint32_t (&o)[8]) {
    o[0] = lo_u16x2(v.x); o[1] = hi_u16x2(v.x); o[2] = lo_u16x2(v.y); o[3] = hi_u16x2(v.y);
    o[4] = lo_u16x2(v.z); o[5] = hi_u16x2(v.z); o[6] = lo_u16x2(v.w); o[7] = hi_u16x2(v.w);
}
__device__ __forceinline__ uint32_t node_e8_unpacked(uint32_t ub, const uint4 &qa, const uint4 &qb, const uint32_t (&mn)[8],
                                                    const uint32_t (&mx)[8]) {
    const uint32_t qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
    uint32_t es = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const uint32_t c2 = min_u16x2(max_u16x2(qv[k], mn[k]), mx[k]);
        es += ld_sh_u8(__byte_perm(c2, ub, 0x7650u) + (2 * k) * CARD);
        es += ld_sh_u8(__byte_perm(c2, ub, 0x7652u) + (2 * k + 1) * CARD);
    }
    return es;
}

// coarse member bound (R17): 8 lookups in the query's [8][256] pair table at cb (256-aligned). P0 / P1
// hold the pair indices of a word: byte k of P0 = hi4(sym_k) | hi4(sym_{k+4}) << 4 (pairs 0..3), byte k
// of P1 = hi4(sym_{8+k}) | hi4(sym_{12+k}) << 4 (pairs 4..7).
__device__ __forceinline__ void pair_index(const uint4 &wv, uint32_t &P0, uint32_t &P1) {
    P0 = ((wv.x >> 4) & 0x0F0F0F0Fu) | (wv.y & 0xF0F0F0F0u);
    P1 = ((wv.z >> 4) & 0x0F0F0F0Fu) | (wv.w & 0xF0F0F0F0u);
}
__device__ __forceinline__ uint32_t coarse_e8(uint32_t cb, uint32_t P0, uint32_t P1) {
    uint32_t a = 0, b = 0;
#pragma unroll
    for (int p = 0; p < 4; p++) a += ld_sh_u8(__byte_perm(P0, cb, 0x7650u | (uint32_t)p) + p * CARD);
#pragma unroll
    for (int p = 0; p < 4; p++) b += ld_sh_u8(__byte_perm(P1, cb, 0x7650u | (uint32_t)p) + (4 + p) * CARD);
    return a + b;
}
__device__ __forceinline__ void st_sh_v4a(uint32_t a, const uint4 &v) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void st_sh_u32a(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_sh_u32(const uint32_t *p) {
    uint32_t r;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return r;
}
__device__ __forceinline__ uint4 ld_sh_v4(const uint4 *p) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return r;
}

__device__ __forceinline__ uint32_t ld_sh_u32a(uint32_t a) {
    uint32_t r;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ uint4 ld_sh_v4a(uint32_t a) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
    return r;
}
// 16-byte global -> shared asynchronous copy (LDGSTS) to a shared-window address
__device__ __forceinline__ void cp_async16_sh(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// 16-byte global -> shared asynchronous copy (LDGSTS); zero-fills the destination when !valid
__device__ __forceinline__ void cp_async16(void *dst_smem, const void *src, bool valid) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst_smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// histogram bin of a kept bound inside its band (for the host's band shrinking)
__device__ __forceinline__ uint32_t hist_bin(float lb, float lo, float hi) {
    const float l0 = fmaxf(lo, 0.f);
    const float span = hi - l0;
    const float x = span > 0.f ? __fdividef(lb - l0, span) : 0.f;
    return min((uint32_t)(fmaxf(x, 0.f) * (float)HIST_BINS), HIST_BINS - 1);
}

struct __align__(16) QConst {  // per query slot, two 16-byte words
    float lo, T;               // band (lo, T]: T = min(band_hi, bsf^2 (1 + delta))
    uint32_t ws, we;           // window [ws, we): already refined, never a candidate
    uint32_t plo, phi;         // the round's position range [plo, phi) (R10; [0, N) unless split)
    uint32_t pad0, pad1;
};

// the keep rule's position part: outside the window, inside the round's range
__device__ __forceinline__ bool pos_ok(const QConst &k, uint32_t pos) {
    return (pos < k.ws || pos >= k.we) && pos >= k.plo && pos < k.phi;
}

__device__ __forceinline__ QConst load_qconst(uint32_t qi, bool valid, const unsigned long long *bsf,
                                              const Band *band, uint32_t slot, const uint32_t *win, float onepd,
                                              bool defer = false) {
    const Band b = valid ? band[slot] : Band{0.f, -1.f, 0u, 0u};
    // hi < 0 encodes a fraction of the BSF threshold (the first band of a query, R15): T = bsf^2 (1 + delta) * -hi
    // (defer: the whole threshold for now; fbdecide_kernel applies the fraction to the costly queries)
    const float tb = bsf_d2(bsf[qi]) * onepd;
    const float tq = valid ? (b.hi < 0.f ? (defer ? tb : tb * -b.hi) : fminf(tb, b.hi)) : -1.0f;  // an invalid slot keeps nothing
    return QConst{b.lo, tq, win[2 * qi], win[2 * qi + 1], b.plo, b.phi, 0u, 0u};
}

// ------------------------------------------------------------------------------------ flat scan
constexpr int LB_THREADS = 256;
constexpr int LB_U = 4;

template <int G>
__global__ void __launch_bounds__(LB_THREADS) lbscan_kernel(const uint4 *__restrict__ sax, uint32_t N,
                                                            const float *__restrict__ lut_all,
                                                            const uint32_t *__restrict__ qmap,
                                                            const Band *__restrict__ band, uint32_t nq,
                                                            const unsigned long long *__restrict__ bsf,
                                                            const uint32_t *__restrict__ win, float onepd,
                                                            uint32_t *__restrict__ cand,
                                                            uint16_t *__restrict__ candq,
                                                            uint32_t *__restrict__ cand_cnt, uint32_t cap,
                                                            uint32_t *__restrict__ hist) {
    extern __shared__ __align__(16) float slut[];  // [G][16][256]
    __shared__ QConst qc[G];
    __shared__ uint32_t qid[G];
    const uint32_t t = threadIdx.x, lane = t & 31;
    const uint32_t g0 = blockIdx.y * G;
    for (uint32_t e = t; e < G * W * CARD; e += LB_THREADS) {
        const uint32_t g = e / (W * CARD);
        const uint32_t qi = g0 + g < nq ? qmap[g0 + g] : qmap[g0];
        slut[e] = lut_all[(uint64_t)qi * W * CARD + (e % (W * CARD))];
    }
    if (t < G) {
        const bool valid = g0 + t < nq;
        const uint32_t qi = valid ? qmap[g0 + t] : qmap[g0];
        qid[t] = qi;
        qc[t] = load_qconst(qi, valid, bsf, band, g0 + t, win, onepd);
    }
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
    const uint64_t step = (uint64_t)gridDim.x * LB_THREADS * LB_U;
    for (uint64_t base = (uint64_t)blockIdx.x * LB_THREADS * LB_U; base < N; base += step) {
        uint4 wv[LB_U];
#pragma unroll
        for (int u = 0; u < LB_U; u++) {
            const uint64_t pos = base + u * LB_THREADS + t;
            wv[u] = pos < N ? ld_stream(sax + pos) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < LB_U; u++) {
            const uint32_t pos = (uint32_t)(base + u * LB_THREADS + t);
            const bool inr = base + u * LB_THREADS + t < N;
#pragma unroll
            for (int g = 0; g < G; g++) {
                const QConst k = qc[g];
                const float lb = word_lb(slut + g * W * CARD, wv[u]);
                const bool keep = inr && lb > k.lo && lb <= k.T && pos_ok(k, pos);
                const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                if (bal) {
                    uint32_t off = 0;
                    if (lane == 0) off = atomicAdd(&cand_cnt[qid[g]], (uint32_t)__popc(bal));
                    off = __shfl_sync(0xffffffffu, off, 0);
                    if (keep) {
                        const uint32_t kk = off + __popc(bal & lt);
                        if (kk < cap) {
                            cand[(uint64_t)qid[g] * cap + kk] = pos;
                            candq[(uint64_t)qid[g] * cap + kk] = 0;  // no bounds recorded: never skipped
                        }
                        atomicAdd(&hist[qid[g] * HIST_BINS + hist_bin(lb, k.lo, k.T)], 1u);
                    }
                }
            }
        }
    }
}

template <int G>
static void launch_g(const isax_index *ix, uint32_t nq, const uint32_t *qmap, const Band *band, float onepd,
                     cudaStream_t s) {
    const size_t smem = (size_t)G * W * CARD * sizeof(float);
    // per launch (the attribute is per device; a failure surfaces as the launch's error)
    cudaFuncSetAttribute(lbscan_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t groups = (nq + G - 1) / G;
    const int per_sm = std::max(1, (int)((227 * 1024) / (smem + 2048)));
    const uint64_t tiles = (ix->N + LB_THREADS * LB_U - 1) / (LB_THREADS * LB_U);
    uint64_t gx = ((uint64_t)sms * per_sm + groups - 1) / groups;
    gx = std::max<uint64_t>(1, umin64(gx, tiles));
    const QueryScratch &qs = ix->qs;
    lbscan_kernel<G><<<dim3((unsigned)gx, groups), LB_THREADS, smem, s>>>(
        reinterpret_cast<const uint4 *>(ix->sax), (uint32_t)ix->N, qs.lut, qmap, band, nq, qs.bsf, qs.win, onepd,
        qs.cand, qs.candq, qs.cand_cnt, qs.cand_cap, qs.cand_hist);
}

// ------------------------------------------------------------------------------------ leaf scan (round 2b, -DISAX_SCAN_V1=1)
// The default scan until round 2c (now nodescan_kernel + itemscan_kernel below; the node bounds and
// the candidate staging defined here are shared): MESSI's node pruning on the sorted array (R11). P:346-349: "the index
// workers traverse the index subtrees ... using BSF to decide which subtrees will be pruned";
// leaves that survive are examined "by first computing lower bound distances using the
// iSAX summaries".
//
// Three node levels: a leaf is LEAF consecutive sorted positions, a super-node SUPER leaves, a
// hyper-node HYPER super-nodes. Inside each super-node the positions follow a kd order (R6b), so
// its leaves are kd cells. A node's summary (leaf_meta_kernel, parent_meta_kernel) is the
// per-segment [min, max] symbol. The node's region on segment s is [beta_min, beta_{max+1}). Its
// MINDIST term is the minimum of LUT[s][c] over c in [min, max]. LUT[s][.] is V-shaped around the
// query's own symbol q_s, so that minimum is LUT[s][clamp(q_s, min, max)]. Every node term is <=
// the term of each member (and of each child node), so a pruned node holds no candidate.
//
// The tests use the u8 tables of scanprep_kernel (R11b): e = floor(LUT * 254 / T), rounded down at
// every step and clamped at 255, so sum_s e <= LB^2 * 254 / T and "sum e > 254" implies LB^2 > T.
// floor is monotone, so a node pruned this way has every member pruned too. Members that pass the
// u8 test get the exact fp32 rule of the flat scan, so the candidate set is exactly the flat scan's
// (tests/test_gpu_parity.py).
//
// Persistent CTAs (two per SM of 512 threads, so one CTA's phase barriers overlap the other's
// work; one of 1024 measured 1-4% slower) pull (query group, chunk of `chunk` leaves) tasks from
// an atomic counter. The u8 tables of the group's G <= 16 queries sit in shared memory.
// Per chunk:
//  A. A0: thread = (hyper-node, query); A1: lane = super-node of a surviving (hyper-node, query);
//     A2: warp iteration = one super-node, lane = one of its 32 leaves, for the queries that kept
//     the super-node (leaf summaries are read only under surviving super-nodes, one iteration
//     ahead). Surviving leaves and their query masks go to a shared worklist; the surviving
//     (leaf, query) pairs are counted per query.
//  B. lane = member: each warp takes one worklist entry per iteration and keeps PD entries in
//     flight in a ring of shared staging slots fed by cp.async (each lane copies and reads only its
//     own word). For every query of the mask it runs the u8 member test (16 lookups), one warp
//     vote, and for the rare survivors the exact rule and the candidate append (one global
//     atomic per warp and query).
constexpr uint32_t LEAF = LEAF_SIZE;
constexpr uint32_t SUPER = SUPER_SIZE / LEAF_SIZE;  // leaves per super-node
constexpr uint32_t HYPER = HYPER_SIZE / SUPER_SIZE; // super-nodes per hyper-node
static_assert(HYPER == 32, "phase A maps the super-nodes of a hyper-node to the lanes of a warp");
static_assert(LEAF == 32 && SUPER == 32, "phase A maps a super-node to a warp iteration and a leaf to a lane");
#ifndef ISAX_COARSE
#define ISAX_COARSE 0
#endif
#if ISAX_COARSE
// the coarse tables (32 KB for 16 queries) and the survivor rings leave room for one CTA per SM
#ifndef ISAX_LF_THREADS
#define ISAX_LF_THREADS 1024
#endif
#ifndef ISAX_LF_CTAS
#define ISAX_LF_CTAS 1
#endif
#endif
#ifndef ISAX_LF_THREADS
#define ISAX_LF_THREADS 512
#endif
constexpr int LF_THREADS = ISAX_LF_THREADS;
#ifndef ISAX_CHUNK
#define ISAX_CHUNK 4096
#endif
#ifndef ISAX_LF_CTAS
#define ISAX_LF_CTAS 2
#endif
constexpr uint32_t CHUNK = ISAX_CHUNK;  // max leaves per phase-A/phase-B round of a CTA
constexpr int LF_CTAS = ISAX_LF_CTAS;   // leaf-scan CTAs per SM
#ifndef ISAX_PD
#define ISAX_PD 2
#endif
constexpr uint32_t PD = ISAX_PD;  // phase B: worklist entries in flight per warp (a power of two)
static_assert((PD & (PD - 1)) == 0, "the staging ring wraps with a mask");
// a u8 member sum <= E_SURE implies LB^2 <= T: sum_s LUT_s * sc < (sum e + 16) / (1 - 2^-23) and
// sc >= (254 / T)(1 - 2^-23), so LB^2 < (237 + 16) / 254 * T * (1 + 2^-20) < T (R11b)
constexpr uint32_t E_SURE = 237;

// Candidate appends ("the data series that are not pruned are stored in a candidate list").
// Each warp stages its kept lanes in a private shared buffer of (position, slot, u8 bound) entries
// (no atomics: the warp's count is a register) and empties it into the global lists itself when it
// holds WB - 32 or more, and at the end of each task: the entries of one query slot get one global
// atomic per flush (match_any groups the lanes by slot). The u8 bound b satisfies b / sc <= LB^2
// (for the refine's skip test). Once a query's list has passed its capacity the slot's flag stops
// this CTA's appends: the list is dropped for the round anyway (R10: an overflowed list is neither
// refined nor needed, only the histogram is), and a query with millions of candidates would
// otherwise serialise every CTA on its count.
#ifndef ISAX_SCAN_V1
#define ISAX_SCAN_V1 0  // 1: the round-2b kernel (leaf worklist, lane = member of a whole leaf), for A/B
#endif
#ifndef ISAX_WB
#define ISAX_WB (ISAX_SCAN_V1 ? 64 : 96)  // (item scan: 0.736 -> 0.728 ms at cfg3 with 96 instead of 48)
#endif
constexpr uint32_t WB = ISAX_WB;  // staged candidates per warp (flushed when more than WB - 32 are staged)
// R17: (member, query) pairs that pass the coarse test wait in a per-warp ring of SV words + metas
// until 32 of them fill one full-test batch (lane = pair)
constexpr uint32_t SV = ISAX_COARSE ? 64 : 0;
constexpr uint32_t CW = ISAX_COARSE ? (W / 2) * CARD : 0;  // coarse table bytes per query
__device__ __forceinline__ void wflush(uint2 *wb, uint32_t &wcnt, uint32_t lane, volatile uint32_t *ovf,
                                       const uint32_t *qid, uint32_t *cand, uint16_t *candq, uint32_t *cand_cnt,
                                       uint32_t cap) {
    __syncwarp();
    for (uint32_t i0 = 0; i0 < wcnt; i0 += 32) {
        const bool have = i0 + lane < wcnt;
        const uint2 en = have ? wb[i0 + lane] : make_uint2(0u, 0u);
        const uint32_t g = have ? (en.y >> 16) : 0xFFFFu;
        const uint32_t peers = __match_any_sync(0xffffffffu, g);
        if (have) {
            const uint32_t leader = __ffs(peers) - 1;
            const uint32_t q = qid[g];
            uint32_t base = 0xffffffffu;
            if (lane == leader && !ovf[g]) {
                const uint32_t c = __popc(peers);
                base = atomicAdd(&cand_cnt[q], c);
                if (base + c > cap) ovf[g] = 1u;
            }
            base = __shfl_sync(peers, base, leader);
            const uint32_t k = base + __popc(peers & ((1u << lane) - 1u));
            ISAX_BOUND(g < 16u);
            if (base != 0xffffffffu && k < cap) {
                cand[(uint64_t)q * cap + k] = en.x;
                candq[(uint64_t)q * cap + k] = (uint16_t)(en.y & 0xFFFFu);
            }
        }
    }
    __syncwarp();
    wcnt = 0;
}

// bq = the candidate's u8 bounds: b | (b2 << 8), b2 that of the second half's segments (R16)
__device__ __forceinline__ void emit(bool keep, uint32_t pos, uint32_t bq, uint32_t g, uint32_t lane, uint32_t lt,
                                     uint2 *wb, uint32_t &wcnt, volatile uint32_t *ovf, const uint32_t *qid,
                                     uint32_t *cand, uint16_t *candq, uint32_t *cand_cnt, uint32_t cap) {
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (!bal || ovf[g]) return;
    if (keep) wb[wcnt + __popc(bal & lt)] = make_uint2(pos, (g << 16) | bq);
    wcnt += __popc(bal);
    if (wcnt > WB - 32) wflush(wb, wcnt, lane, ovf, qid, cand, candq, cand_cnt, cap);
}

// u8 table entry (R11b): floor(v * sc) with sc = 254 / T rounded down, clamped at 255. v = 0 maps
// to 0, so T = 0 (an exact duplicate in the window) keeps exactly the members with LB^2 = 0.
__device__ __forceinline__ uint32_t q8(float v, float sc) {
    if (!(v > 0.f)) return 0u;
    const float x = __fmul_rd(v, sc);
    return x >= 255.f ? 255u : (uint32_t)x;
}

// Per active slot of a scan launch: its constants (band lo, T, window) and its u8 table, once,
// instead of in every CTA that takes one of its tasks. One CTA per slot.
__global__ void __launch_bounds__(256) scanprep_kernel(const float *__restrict__ lut_all, const uint32_t *__restrict__ qmap,
                                                       const Band *__restrict__ band,
                                                       const unsigned long long *__restrict__ bsf,
                                                       const uint32_t *__restrict__ win, float onepd,
                                                       uint8_t *__restrict__ lut8, uint8_t *__restrict__ lut8c,
                                                       uint4 *__restrict__ qconst,
                                                       float *__restrict__ qscale, float *__restrict__ qT,
                                                       unsigned long long *__restrict__ bsf_scan, uint32_t B,
                                                       uint32_t *__restrict__ cand_cnt, uint32_t *__restrict__ cand_cnt2,
                                                       uint32_t *__restrict__ cnt_hi, uint32_t *__restrict__ cnt_f,
                                                       uint32_t *__restrict__ hist, uint32_t *__restrict__ task_ctr,
                                                       uint32_t *__restrict__ ctl, uint32_t nctl, uint32_t *__restrict__ qkept,
                                                       bool defer) {
    const uint32_t i = blockIdx.x;
    // the launch's counters: every batch slot's candidate counts (block 0), the scanned query's
    // histogram (its block), the persistent scan's task counter
    if (i == 0) {
        for (uint32_t q = threadIdx.x; q < B; q += blockDim.x) cand_cnt[q] = cand_cnt2[q] = cnt_hi[q] = cnt_f[q] = 0;
        if (threadIdx.x == 0) *task_ctr = 0;
        for (uint32_t k = threadIdx.x; k < nctl; k += blockDim.x) ctl[k] = 0;  // the item scan's per-group words
    }
    if (threadIdx.x < HIST_BINS) hist[qmap[i] * HIST_BINS + threadIdx.x] = 0;
    const uint32_t qi = qmap[i];
    if (threadIdx.x == 0) qkept[i] = 0;  // super-nodes the node scan keeps for this slot
    const QConst k = load_qconst(qi, true, bsf, band, i, win, onepd, defer);
    if (threadIdx.x == 0) {
        qconst[2 * i] = make_uint4(__float_as_uint(k.lo), __float_as_uint(k.T), k.ws, k.we);
        qconst[2 * i + 1] = make_uint4(k.plo, k.phi, 0u, 0u);
    }
    const bool none = !(k.T >= 0.f);  // an empty band keeps nothing
    const float sc = none ? 0.f : __fdiv_rd(254.0f, k.T);  // T = 0 -> +inf
    if (threadIdx.x == 0) {
        qscale[qi] = sc;
        qT[qi] = k.T;
        // the BSF the scan uses; the id's lowest bit tells the host whether a first-band slot really
        // got the fraction (always, unless fbdecide_kernel decides per query)
        bsf_scan[qi] = (bsf[qi] & ~1ull) | (defer ? 0ull : 1ull);
    }
    const float4 *L = reinterpret_cast<const float4 *>(lut_all + (uint64_t)qi * W * CARD);
    uint32_t *o = reinterpret_cast<uint32_t *>(lut8 + (uint64_t)i * W * CARD);
    for (uint32_t e = threadIdx.x; e < W * CARD / 4; e += blockDim.x) {
        const float4 v = __ldg(L + e);
        o[e] = none ? 0xFFFFFFFFu : (q8(v.x, sc) | q8(v.y, sc) << 8 | q8(v.z, sc) << 16 | q8(v.w, sc) << 24);
    }
    // the coarse table (R17): per segment and high nibble a, the smallest entry of its 16 symbols
    // (q8 is monotone, so that is the entry of the smallest LUT value); then per segment pair
    // (s1, s2) = (p, p + 4) for p < 4, (p + 4, p + 8) for p >= 4, entry a | b << 4 =
    // min(255, mn[s1][a] + mn[s2][b]) <= e[s1][c1] + e[s2][c2] for every c1 >> 4 = a, c2 >> 4 = b.
    __shared__ uint32_t mn[W][16];
    {
        const uint32_t sg = threadIdx.x >> 4, a = threadIdx.x & 15u;  // 256 threads = 16 x 16
        const float *Ls = lut_all + (uint64_t)qi * W * CARD + sg * CARD + 16 * a;
        float v = __ldg(Ls);
#pragma unroll
        for (int c = 1; c < 16; c++) v = fminf(v, __ldg(Ls + c));
        mn[sg][a] = none ? 255u : q8(v, sc);
    }
    __syncthreads();
    uint32_t *oc = reinterpret_cast<uint32_t *>(lut8c + (uint64_t)i * (W / 2) * CARD);
    for (uint32_t e = threadIdx.x; e < (W / 2) * CARD / 4; e += blockDim.x) {
        const uint32_t p = e >> 6, s1 = p < 4 ? p : p + 4, s2 = s1 + 4;
        uint32_t word = 0;
#pragma unroll
        for (uint32_t k = 0; k < 4; k++) {
            const uint32_t idx = (e & 63u) * 4 + k, a = idx & 15u, b = idx >> 4;
            word |= min(255u, mn[s1][a] + mn[s2][b]) << (8 * k);
        }
        oc[e] = word;
    }
}

// R15, per query: after the node scan ran under the whole window threshold, a first-band slot whose
// query kept more than `heavy` super-nodes (a costly scan: its window probably missed the near
// neighbour) gets the first band after all: T = bsf^2 (1 + delta) * -band.hi, with its u8 table
// and constants rewritten for it. Its entries stay (super-nodes kept under the larger threshold: a
// superset, tested again at the leaf level). The other first-band slots keep the whole threshold
// and are done in this round. One CTA per slot.
__global__ void __launch_bounds__(256) fbdecide_kernel(const float *__restrict__ lut_all, const uint32_t *__restrict__ qmap,
                                                       const Band *__restrict__ band, const unsigned long long *__restrict__ bsf,
                                                       float onepd, const uint32_t *__restrict__ qkept, uint32_t heavy,
                                                       uint8_t *__restrict__ lut8, uint4 *__restrict__ qconst,
                                                       float *__restrict__ qscale, float *__restrict__ qT,
                                                       unsigned long long *__restrict__ bsf_scan) {
    const uint32_t i = blockIdx.x, qi = qmap[i];
    const Band b = band[i];
    if (!(b.hi < 0.f) || qkept[i] <= heavy) return;  // (uniform per CTA)
    const float T = bsf_d2(bsf[qi]) * onepd * -b.hi;
    const bool none = !(T >= 0.f);
    const float sc = none ? 0.f : __fdiv_rd(254.0f, T);
    if (threadIdx.x == 0) {
        uint4 k = qconst[2 * i];
        k.y = __float_as_uint(T);
        qconst[2 * i] = k;
        qscale[qi] = sc;
        qT[qi] = T;
        bsf_scan[qi] |= 1ull;
    }
    const float4 *L = reinterpret_cast<const float4 *>(lut_all + (uint64_t)qi * W * CARD);
    uint32_t *o = reinterpret_cast<uint32_t *>(lut8 + (uint64_t)i * W * CARD);
    for (uint32_t e = threadIdx.x; e < W * CARD / 4; e += blockDim.x) {
        const float4 v = __ldg(L + e);
        o[e] = none ? 0xFFFFFFFFu : (q8(v.x, sc) | q8(v.y, sc) << 8 | q8(v.z, sc) << 16 | q8(v.w, sc) << 24);
    }
}

template <int G>
__global__ void __launch_bounds__(LF_THREADS, LF_CTAS) leafscan_kernel(
    const uint4 *__restrict__ sax, const uint8_t *__restrict__ lmeta, const uint8_t *__restrict__ smeta,
    const uint8_t *__restrict__ hmeta, uint32_t N, const float *__restrict__ lut_all, const uint8_t *__restrict__ lut8_all,
    const uint8_t *__restrict__ lut8c_all, const uint4 *__restrict__ qconst_all,
    const uint8_t *__restrict__ qsax_all, const uint32_t *__restrict__ qmap, uint32_t nq, uint32_t nleaf,
    uint32_t chunk, uint32_t *__restrict__ cand, uint16_t *__restrict__ candq, uint32_t *__restrict__ cand_cnt, uint32_t cap,
    uint32_t *__restrict__ hist, uint32_t *__restrict__ leaves_alive, unsigned long long *__restrict__ scan_bytes_dev,
    uint32_t *__restrict__ task_ctr, uint32_t run) {
    // shared: [G][16][256] u8 tables | [CHUNK] worklist | [NW][PD][LEAF] staged words
    // (the dynamic region follows the static variables, so the u8 tables are aligned by hand: the
    // PRMT address trick needs a 256-aligned base)
    extern __shared__ __align__(16) uint8_t smem_dyn[];
    const uint32_t raw8 = (uint32_t)__cvta_generic_to_shared(smem_dyn);
    const uint32_t lut8_sh = (raw8 + 255u) & ~255u;
    uint8_t *lut8 = smem_dyn + (lut8_sh - raw8);
    constexpr uint32_t NW = LF_THREADS / 32;
    const uint32_t lut8c_sh = lut8_sh + G * W * CARD;  // [G][8][256] coarse tables (R17; CW = 0 without)
    uint32_t *worklist = reinterpret_cast<uint32_t *>(lut8 + G * (W * CARD + CW));  // (leaf offset in chunk) | (query mask << 16)
    const uint32_t wl_sh = lut8_sh + G * (W * CARD + CW);
    const uint32_t stage_sh = wl_sh + CHUNK * 4;  // 16-byte aligned
    uint2 *wbuf = reinterpret_cast<uint2 *>(worklist + CHUNK + NW * PD * LEAF * 4) + (threadIdx.x >> 5) * WB;  // this warp's staged candidates
    // this warp's survivor ring (R17): SV words, then SV metas (member offset in the chunk | slot << 20)
    const uint32_t sv_sh = wl_sh + CHUNK * 4 + NW * PD * LEAF * 16 + NW * WB * 8 + (threadIdx.x >> 5) * SV * 20;
    uint32_t wcnt = 0;
    __shared__ QConst qc[G];
    __shared__ uint4 qsym[G][2];  // the query's 16 symbols as 8 u16x2 pairs
    __shared__ uint32_t qid[G], alive_cnt[G], s_ovf[G];
    __shared__ float qsc[G];  // 254 / T rounded down (the u8 table scale)
    __shared__ uint32_t shist[G][HIST_BINS];
    __shared__ uint32_t wl_cnt, s_task;
    __shared__ uint32_t hmask[CHUNK / (SUPER * HYPER) + 1];  // query mask of each hyper-node of the chunk
    __shared__ uint32_t smask_sh[CHUNK / SUPER];            // query mask of each super-node of the chunk
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    constexpr uint32_t FULL = 0xffffffffu;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t nchunks = (nleaf + chunk - 1) / chunk;
    const uint32_t ngroups = (nq + G - 1) / G;
    const uint32_t ntasks = nchunks * ngroups;
    const uint4 *meta4 = reinterpret_cast<const uint4 *>(lmeta);
    const uint4 *smeta4 = reinterpret_cast<const uint4 *>(smeta);
    const uint4 *hmeta4 = reinterpret_cast<const uint4 *>(hmeta);
    uint32_t bytes = 0;            // node summaries and words this thread read
    uint32_t my_alive = 0;         // lane g < G: loaded (leaf, query g) pairs of this warp
    uint32_t g0 = 0xffffffffu;     // first query slot of the group whose tables are loaded
    // the loaded group's histograms and surviving-leaf counts into global memory
    auto flush = [&]() {
        if (lane < G && my_alive) atomicAdd(&alive_cnt[lane], my_alive);
        my_alive = 0;
        __syncthreads();
        if (t < G && alive_cnt[t] && g0 + t < nq) atomicAdd(&leaves_alive[qid[t]], alive_cnt[t]);
        for (uint32_t e = t; e < G * HIST_BINS; e += LF_THREADS) {
            const uint32_t g = e / HIST_BINS, b = e % HIST_BINS;
            if (g0 + g < nq && shist[g][b]) atomicAdd(&hist[qid[g] * HIST_BINS + b], shist[g][b]);
        }
        __syncthreads();
    };
    // tasks are taken in runs of `run` consecutive ones (launch_leaf: 1)
    __shared__ uint32_t s_next, s_end;
    if (t == 0) {
        wl_cnt = 0;
        s_next = s_end = 0;
    }
    for (;;) {
        if (t == 0) {
            if (s_next >= s_end) {
                s_next = atomicAdd(task_ctr, run);
                s_end = s_next + run;
            }
            s_task = s_next++;
        }
        __syncthreads();
        const uint32_t task = s_task;
        if (task >= ntasks) break;
        const uint32_t grp = task / nchunks, ch = task % nchunks;
        if (grp * G != g0) {  // new query group: load its tables and constants
            if (g0 != 0xffffffffu) flush();
            g0 = grp * G;
            for (uint32_t e = t; e < G * HIST_BINS; e += LF_THREADS) shist[e / HIST_BINS][e % HIST_BINS] = 0;
            if (t < G) {
                const bool valid = g0 + t < nq;
                const uint32_t slot = valid ? g0 + t : g0;
                const uint32_t qi = qmap[slot];
                qid[t] = qi;
                alive_cnt[t] = 0;
                s_ovf[t] = 0;
                const uint4 w = reinterpret_cast<const uint4 *>(qsax_all)[qi];
                qsym[t][0] = make_uint4(lo_u16x2(w.x), hi_u16x2(w.x), lo_u16x2(w.y), hi_u16x2(w.y));
                qsym[t][1] = make_uint4(lo_u16x2(w.z), hi_u16x2(w.z), lo_u16x2(w.w), hi_u16x2(w.w));
                const uint4 k = qconst_all[2 * slot], k2 = qconst_all[2 * slot + 1];
                qc[t] = valid ? QConst{__uint_as_float(k.x), __uint_as_float(k.y), k.z, k.w, k2.x, k2.y, 0u, 0u}
                              : QConst{0.f, -1.f, 0u, 0u, 0u, 0u, 0u, 0u};
                qsc[t] = valid && __uint_as_float(k.y) >= 0.f ? __fdiv_rd(254.0f, __uint_as_float(k.y)) : 0.f;  // as scanprep
            }
            // the group's u8 tables; a padding slot gets all-255 entries (it prunes everything)
            {
                const uint4 *src = reinterpret_cast<const uint4 *>(lut8_all + (uint64_t)g0 * W * CARD);
                uint4 *dst = reinterpret_cast<uint4 *>(lut8);
                constexpr uint32_t PER = W * CARD / 16;
                for (uint32_t e = t; e < G * PER; e += LF_THREADS)
                    dst[e] = g0 + e / PER < nq ? __ldg(src + e) : make_uint4(FULL, FULL, FULL, FULL);
#if ISAX_COARSE
                const uint4 *srcc = reinterpret_cast<const uint4 *>(lut8c_all + (uint64_t)g0 * CW);
                uint4 *dstc = reinterpret_cast<uint4 *>(lut8 + G * W * CARD);
                constexpr uint32_t PERC = CW / 16;
                for (uint32_t e = t; e < G * PERC; e += LF_THREADS)
                    dstc[e] = g0 + e / PERC < nq ? __ldg(srcc + e) : make_uint4(FULL, FULL, FULL, FULL);
#endif
            }
            __syncthreads();
        }
        const uint32_t c0 = ch * chunk;  // a multiple of SUPER
        const uint32_t c1 = min(c0 + chunk, nleaf);
        // ---- phase A: three node levels, top down.
        const uint32_t s0 = c0 / SUPER, send = (c1 + SUPER - 1) / SUPER;  // the chunk's super-nodes
        const uint32_t h0 = s0 / HYPER, nh = (send - 1) / HYPER - h0 + 1;  // its hyper-nodes (<= 8)
        for (uint32_t e = t; e < send - s0; e += LF_THREADS) smask_sh[e] = 0;
        if (t < nh) hmask[t] = 0;
        __syncthreads();
        // A0: thread = (hyper-node, query). A hyper-node may extend beyond the chunk (chunk of 512
        // leaves): its bound is over a superset of the chunk's positions, still a lower bound.
        if (t < nh * 16u) {
            const uint32_t h = t >> 4, g = t & 15u;
            if (g < G) {
                const uint4 a = __ldg(hmeta4 + 2 * (uint64_t)(h0 + h)), b = __ldg(hmeta4 + 2 * (uint64_t)(h0 + h) + 1);
                if (node_e8(lut8_sh + g * W * CARD, qsym[g][0], qsym[g][1], a, b) <= 254u) atomicOr(&hmask[h], 1u << g);
                bytes += 32;
            }
        }
        __syncthreads();
#ifndef ISAX_NO_EARLY
        {  // a chunk whose hyper-nodes are pruned for every query of the group: the next task
            uint32_t any = 0;
            for (uint32_t h = 0; h < nh; h++) any |= hmask[h];
            if (!any) continue;  // (uniform; wl_cnt is still 0)
        }
#endif
        // A1: for each (hyper-node, query) that survived, lane = one of its 32 super-nodes
        for (uint32_t pr = warp; pr < nh * 16u; pr += NW) {
            const uint32_t h = pr >> 4, g = pr & 15u;
            if (!((hmask[h] >> g) & 1u)) continue;
            const uint32_t sn = (h0 + h) * HYPER + lane;
            if (sn >= s0 && sn < send) {
                bytes += 32;
                const uint4 a = __ldg(smeta4 + 2 * (uint64_t)sn), b = __ldg(smeta4 + 2 * (uint64_t)sn + 1);
                if (node_e8(lut8_sh + g * W * CARD, qsym[g][0], qsym[g][1], a, b) <= 254u)
                    atomicOr(&smask_sh[sn - s0], 1u << g);
            }
        }
        __syncthreads();
        // A2: warp iteration = one super-node (s0 + warp + NW j), lane = one of its 32 leaves, for
        // the queries that kept the super-node (a rolled loop over the mask's bits). Leaf summaries
        // are read only under surviving super-nodes, one iteration ahead.
        const uint4 *meta8 = meta4;
        constexpr uint32_t MW = 2;
        uint32_t nmask = 0;
        uint4 mn_n = make_uint4(0, 0, 0, 0), mx_n = mn_n;
        if (s0 + warp < send) {
            nmask = smask_sh[warp];
            const uint32_t leaf = (s0 + warp) * SUPER + lane;
            if (nmask && leaf < c1) {
                mn_n = __ldg(meta8 + MW * (uint64_t)leaf);
                mx_n = __ldg(meta8 + MW * (uint64_t)leaf + 1);
            }
        }
        for (uint32_t sn = s0 + warp; sn < send; sn += NW) {
            const uint32_t leaf = sn * SUPER + lane;
            const uint32_t cur_mask = nmask;
            const uint4 mn4 = mn_n, mx4 = mx_n;
            if (sn + NW < send) {
                nmask = smask_sh[sn + NW - s0];
                const uint32_t l2 = leaf + NW * SUPER;
                if (nmask && l2 < c1) {
                    mn_n = __ldg(meta8 + MW * (uint64_t)l2);
                    mx_n = __ldg(meta8 + MW * (uint64_t)l2 + 1);
                }
            }
            if (!cur_mask) continue;  // the whole super-node is pruned for every query
            const bool inr = leaf < c1;
            if (inr) bytes += 32;
            uint32_t alive = 0;
#pragma unroll 1
            for (uint32_t mm = cur_mask; mm; mm &= mm - 1) {
                const uint32_t g = __ffs(mm) - 1;
                const bool ok = inr && node_e8(lut8_sh + g * W * CARD, qsym[g][0], qsym[g][1], mn4, mx4) <= 254u;
                alive |= (ok ? 1u : 0u) << g;
                // (leaf, query g) pairs that phase B will test, counted by lane g (stats)
                const uint32_t np = __popc(__ballot_sync(FULL, ok));
                if (lane == (uint32_t)g) my_alive += np;
            }
            const uint32_t bal = __ballot_sync(FULL, alive != 0);
            if (bal) {
                uint32_t off = 0;
                if (lane == 0) off = atomicAdd(&wl_cnt, (uint32_t)__popc(bal));
                off = __shfl_sync(FULL, off, 0);
                ISAX_BOUND(off + __popc(bal) <= CHUNK && leaf - c0 < 0x10000u);
                if (alive) worklist[off + __popc(bal & lt)] = (leaf - c0) | (alive << 16);
            }
        }
        __syncthreads();
        // ---- phase B: the members of surviving leaves, one worklist entry per warp iteration
        // (lane = member). Each warp takes entries warp, warp + NW, ... and keeps PD of them in
        // flight in its own ring of shared staging slots (cp.async, one commit group per entry).
        // A lane copies and reads only its own word, so no warp barrier is needed. The sorted SAX
        // array is padded to whole leaves (api.cu), so the loads need no bounds test. Addresses are
        // shared-window offsets (u32), the ring position a byte offset wrapped with a mask.
        const uint32_t nwl = wl_cnt;
        if (t == 0) bytes += nwl * LEAF * 16u;  // the worklist leaves' words (a partial last leaf is counted whole)
        constexpr uint32_t SLOT = LEAF * 16;  // bytes of one staged leaf
        const uint32_t ring = stage_sh + warp * PD * SLOT + lane * 16;
        const char *gsrc = reinterpret_cast<const char *>(sax + (uint64_t)c0 * LEAF + lane);
        uint32_t pf = warp, pfo = 0;  // next entry to prefetch, its ring offset
#pragma unroll
        for (uint32_t k = 0; k < PD - 1; k++) {
            if (pf < nwl) cp_async16_sh(ring + pfo, gsrc + (size_t)(ld_sh_u32a(wl_sh + 4 * pf) & 0xFFFFu) * SLOT);
            cp_async_commit();
            pf += NW;
            pfo = (pfo + SLOT) & (PD * SLOT - 1);
        }
        uint32_t co = 0;  // ring offset of the entry being consumed
#if ISAX_COARSE
        // R17: the full member test (below) runs on batches of 32 (member, query) pairs that passed
        // the coarse test, one pair per lane; the survivors of a batch get the exact rule and emit.
        uint32_t sv_head = 0, sv_tail = 0;  // warp-uniform ring positions
        auto full_batch = [&](uint32_t cnt) {
            __syncwarp();
            const bool have = lane < cnt;
            const uint32_t ri = (sv_head + lane) & (SV - 1u);
            const uint4 wv = have ? ld_sh_v4a(sv_sh + ri * 16u) : make_uint4(0u, 0u, 0u, 0u);
            const uint32_t m = have ? ld_sh_u32a(sv_sh + SV * 16u + ri * 4u) : 0u;
            __syncwarp();
            sv_head += cnt;
            const uint32_t g = m >> 20;
            uint32_t e8hi;
            const uint32_t e8 = word_e8(lut8_sh + g * W * CARD, wv, e8hi);
            const bool maybe = have && e8 <= 254u;
            if (!__any_sync(FULL, maybe)) return;
            // the keep rule, as in the per-query loop without R17 (see there)
            const uint32_t pos = c0 * LEAF + (m & 0xFFFFFu);
            const QConst kq = qc[g];
            const bool band0 = kq.lo < 0.f;
            const bool first = maybe && band0;
            const bool check = maybe && !band0;
            const float lb = check ? word_lb(lut_all + (uint64_t)qid[g] * W * CARD, wv) : 0.f;
            const bool keep = (first || (check && lb > kq.lo && lb <= kq.T)) && pos_ok(kq, pos);
            uint32_t b = e8 <= E_SURE ? e8 : B_UNCHECKED;
            if (check) {
                const float y = __fmul_rd(lb, qsc[g]);
                b = lb > 0.f ? (y >= 254.f ? 254u : (uint32_t)y) : 0u;
            }
            if (keep) atomicAdd(&shist[g][first ? min(e8 * HIST_BINS / 254u, HIST_BINS - 1) : hist_bin(lb, kq.lo, kq.T)], 1u);
            // lanes of several slots: a slot whose list overflowed stops appending (as emit)
            ISAX_BOUND(!keep || pos < N);
            const bool k2 = keep && !s_ovf[g];
            const uint32_t bal = __ballot_sync(FULL, k2);
            if (!bal) return;
            if (k2) wbuf[wcnt + __popc(bal & lt)] = make_uint2(pos, (g << 16) | b | (e8hi << 8));
            wcnt += __popc(bal);
            if (wcnt > WB - 32) wflush(wbuf, wcnt, lane, s_ovf, qid, cand, candq, cand_cnt, cap);
        };
#endif
        for (uint32_t e = warp; e < nwl; e += NW) {
            if (pf < nwl) cp_async16_sh(ring + pfo, gsrc + (size_t)(ld_sh_u32a(wl_sh + 4 * pf) & 0xFFFFu) * SLOT);
            cp_async_commit();
            pf += NW;
            pfo = (pfo + SLOT) & (PD * SLOT - 1);
            cp_async_wait<PD - 1>();
            const uint32_t ent = ld_sh_u32a(wl_sh + 4 * e);
            const uint32_t wp = ring + co;
            const uint4 wv = ld_sh_v4a(wp);
            co = (co + SLOT) & (PD * SLOT - 1);
#if ISAX_COARSE
            // coarse test per query of the mask (8 lookups, R17); passing pairs join the ring
            const uint32_t memb = (ent & 0xFFFFu) * LEAF + lane;  // member offset in the chunk
            const bool inN = c0 * LEAF + memb < N;
            uint32_t P0, P1;
            pair_index(wv, P0, P1);
#pragma unroll 1
            for (uint32_t mm = ent >> 16; mm; mm &= mm - 1) {
                const uint32_t g = __ffs(mm) - 1;
                const bool pass = inN && coarse_e8(lut8c_sh + g * CW, P0, P1) <= 254u;
                const uint32_t bal = __ballot_sync(FULL, pass);
                if (!bal) continue;
                ISAX_BOUND(sv_tail - sv_head + __popc(bal) <= SV);
                if (pass) {
                    const uint32_t ri = (sv_tail + __popc(bal & lt)) & (SV - 1u);
                    st_sh_v4a(sv_sh + ri * 16u, wv);
                    st_sh_u32a(sv_sh + SV * 16u + ri * 4u, memb | (g << 20));
                }
                sv_tail += __popc(bal);
                if (sv_tail - sv_head >= 32u) full_batch(32u);
            }
#else
            // rolled loop over the queries that kept the leaf: unrolling it over G made the
            // kernel ~120 KB of SASS, and instruction-cache misses became the top stall
#pragma unroll 1
            for (uint32_t mm = ent >> 16; mm; mm &= mm - 1) {
                const uint32_t g = __ffs(mm) - 1;
                // integer member filter: 16 lookups of 2.5 instructions (PRMT address, LDS.U8, half
                // an IADD3)
                uint32_t e8hi;
                const uint32_t e8 = word_e8(lut8_sh + g * W * CARD, wv, e8hi);
                if (!__any_sync(FULL, e8 <= 254u)) continue;
                // The flat scan's rule is lo < LB^2 <= T on the exact fp32 bound. A u8 sum <= E_SURE
                // already implies LB^2 <= T (R11b), and in the first band (lo < 0) lo < LB^2 always
                // holds. In the first band, members with a u8 sum in (E_SURE, 254] are kept marked
                // B_UNCHECKED and get the exact rule in candcheck_kernel, many at a time; in later
                // bands every member gets it here. A first-band member's histogram bin comes from
                // its u8 sum, never above its exact bin (band shrinking, R10, stays an upper bound
                // on the count).
                const uint32_t pos = (c0 + (ent & 0xFFFFu)) * LEAF + lane;
                const bool maybe = pos < N && e8 <= 254u;
                const QConst kq = qc[g];
                const bool band0 = kq.lo < 0.f;
                const bool first = maybe && band0;
                const bool check = maybe && !band0;
                // the word is re-read here (volatile), so that the compiler does not hoist the fp32
                // path's address arithmetic out of the query loop into every entry
                const float lb = check ? word_lb(lut_all + (uint64_t)qid[g] * W * CARD, ld_sh_v4a(wp)) : 0.f;
                const bool keep = (first || (check && lb > kq.lo && lb <= kq.T)) && pos_ok(kq, pos);
                // the candidate's u8 bound b <= LB^2 * sc (for the refine), or B_UNCHECKED
                uint32_t b = e8 <= E_SURE ? e8 : B_UNCHECKED;
                if (check) {
                    const float y = __fmul_rd(lb, qsc[g]);
                    b = lb > 0.f ? (y >= 254.f ? 254u : (uint32_t)y) : 0u;
                }
                if (keep)
                    atomicAdd(&shist[g][first ? min(e8 * HIST_BINS / 254u, HIST_BINS - 1) : hist_bin(lb, kq.lo, kq.T)], 1u);
                ISAX_BOUND(!keep || pos < N);
                emit(keep, pos, b | (e8hi << 8), g, lane, lt, wbuf, wcnt, s_ovf, qid, cand, candq, cand_cnt, cap);
            }
#endif
        }
#if ISAX_COARSE
        if (sv_tail != sv_head) full_batch(sv_tail - sv_head);  // the task's last pairs (warp-uniform)
#endif
        if (wcnt) wflush(wbuf, wcnt, lane, s_ovf, qid, cand, candq, cand_cnt, cap);  // (warp-uniform)
        cp_async_wait<0>();  // the trailing (empty) groups
        __syncthreads();
        if (t == 0) wl_cnt = 0;
    }
    if (g0 != 0xffffffffu) flush();
    bytes = __reduce_add_sync(FULL, bytes);
    if (lane == 0 && bytes) atomicAdd(scan_bytes_dev, (unsigned long long)bytes);
}

// ------------------------------------------------------------------------------------ node scan + item scan
// (R11c) The default scan since round 2c, two kernels.
//
// Why: under a surviving leaf most members still fail (about 2% pass at config 3), because a
// 32-row box is loose in 16 dimensions. One more node level, the kd cells of KD_CELL = 8 rows (the
// last two kd levels of superkd_kernel), removes about half of the member tests
// (tools/offline_readings.py `sub`: 0.52-0.54 of the members lie under surviving cells). To turn
// that into fewer instructions the member tests are pair-major: a warp iteration tests four
// surviving (cell, query) pairs, one per quarter warp, instead of the 32 members of one leaf. And
// the v1 kernel spent a third of its time in per-task fixed costs (the hyper- and super-node
// phases and their barriers, once per chunk and query group: halving the group size added 0.28 ms
// at config 3), so the upper node levels moved to a kernel of their own.
//
// nodescan_kernel: warp = hyper-node, for the 16 queries of a group: the hyper-node bound (lane =
//   query), then for every query that kept it the bounds of its 32 super-nodes (lane = super-node).
//   Output per group: a list of entries (super-node, mask of the queries that kept it), appended
//   with one global atomic per warp and hyper-node, and the group's work estimate (kept pairs).
// itemscan_kernel: persistent CTAs (the group's 16 u8 tables in shared memory); CTAs spread over
//   the groups in proportion to their work and move on when a group's list runs out. Each warp
//   claims entries from the group's cursor and runs everything below by itself, in registers and a
//   few hundred bytes of its own shared memory, with no CTA barrier:
//     A2  per entry: lane = one of the super-node's 32 leaves (summaries loaded once), one node
//         bound per query of the mask -> items (super-node, query, alive-leaf mask) in a ring;
//     A3  per item: lane = one of the 4 cells of an alive leaf, 32 cells per iteration: node bound
//         -> the item's alive cells (a byte list);
//     B   per item: quarter warp = one alive cell, lane = one of its 8 members: the u8 member test
//         (16 lookups), a vote, and the rare path of the pairs that pass (exact rule, histogram,
//         append).
//   A3 of the next item runs before B of this one, the next entry is claimed and its leaf
//   summaries prefetched into L2 an entry ahead, and the cell summaries of alive leaves and the
//   words of alive cells are prefetched into L2 as soon as they are known.
constexpr uint32_t CELL = KD_CELL;
constexpr uint32_t CPL = LEAF / CELL;        // cells per leaf
constexpr uint32_t CPS = SUPER_SIZE / CELL;  // cells per super-node
static_assert(CPL == 4 && CPS == 128, "A3 maps four cells of a leaf to four lanes; a cell index is 7 bits");
constexpr uint32_t CLIST = CPS + 8;          // bytes of an alive-cell list: a cell index each, 8 padding entries
constexpr uint32_t IQ = 32;                  // item ring slots per warp (a power of two; an entry adds at most 16)
constexpr uint32_t WSC = 32 + 2 * CLIST + IQ * 8;  // per-warp scratch bytes: alive-leaf list, two alive-cell lists, item ring
// scan control words in qs.scan_ctl (reset by scanprep_kernel): per group its entry count, its
// claim cursor and its work estimate
constexpr uint32_t CTL_CNT = 0, CTL_CUR = 1, CTL_WORK = 2, CTL_CNT_L = 3, CTL_WORDS = 4;
// entries kept by HEAVY or more queries are stored from the front of the group's array and claimed
// first, the others from the back and last: the entries still in flight when a list runs out are
// then the short ones (0 = one list in arrival order)
#ifndef ISAX_HEAVY
#define ISAX_HEAVY 0
#endif
constexpr uint32_t HEAVY = ISAX_HEAVY;

__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
__device__ __forceinline__ void st_sh_u8a(uint32_t a, uint32_t v) { asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
__device__ __forceinline__ void st_sh_v2a(uint32_t a, uint32_t x, uint32_t y) {
    asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(a), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ uint2 ld_sh_v2a(uint32_t a) {
    uint2 r;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(a));
    return r;
}

// the group's u8 tables, query symbols and constants into shared memory (both kernels)
template <int G, int THREADS>
__device__ __forceinline__ void load_group(uint32_t g0, uint32_t nq, const uint32_t *__restrict__ qmap,
                                           const uint8_t *__restrict__ qsax_all, const uint8_t *__restrict__ lut8_all,
                                           uint8_t *lut8, uint4 (*qsym)[2], uint32_t *qid) {
    const uint32_t t = threadIdx.x;
    if (t < G) {
        const uint32_t slot = g0 + t < nq ? g0 + t : g0;
        const uint32_t qi = qmap[slot];
        qid[t] = qi;
        const uint4 w = reinterpret_cast<const uint4 *>(qsax_all)[qi];
        qsym[t][0] = make_uint4(lo_u16x2(w.x), hi_u16x2(w.x), lo_u16x2(w.y), hi_u16x2(w.y));
        qsym[t][1] = make_uint4(lo_u16x2(w.z), hi_u16x2(w.z), lo_u16x2(w.w), hi_u16x2(w.w));
    }
    // a padding slot gets all-255 entries (it prunes everything)
    const uint4 *src = reinterpret_cast<const uint4 *>(lut8_all + (uint64_t)g0 * W * CARD);
    uint4 *dst = reinterpret_cast<uint4 *>(lut8);
    constexpr uint32_t PER = W * CARD / 16;
    for (uint32_t e = t; e < G * PER; e += THREADS)
        dst[e] = g0 + e / PER < nq ? __ldg(src + e) : make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
}

constexpr int NS_THREADS = 256;
template <int G>
__global__ void __launch_bounds__(NS_THREADS) nodescan_kernel(
    const uint8_t *__restrict__ smeta, const uint8_t *__restrict__ hmeta, uint32_t nsuper, uint32_t nhyper,
    const uint8_t *__restrict__ lut8_all, const uint8_t *__restrict__ qsax_all, const uint32_t *__restrict__ qmap, uint32_t nq,
    uint32_t hyper_per_cta, uint2 *__restrict__ entries, uint32_t *__restrict__ ctl,
    unsigned long long *__restrict__ scan_bytes_dev, uint32_t *__restrict__ qkept, bool count_only) {
    extern __shared__ __align__(16) uint8_t smem_dyn[];
    const uint32_t raw8 = (uint32_t)__cvta_generic_to_shared(smem_dyn);
    const uint32_t lut8_sh = (raw8 + 255u) & ~255u;
    uint8_t *lut8 = smem_dyn + (lut8_sh - raw8);
    __shared__ uint4 qsym[G][2];
    __shared__ uint32_t qid[G];
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    constexpr uint32_t FULL = 0xffffffffu, NW = NS_THREADS / 32;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t grp = blockIdx.y, g0 = grp * G;
    load_group<G, NS_THREADS>(g0, nq, qmap, qsax_all, lut8_all, lut8, qsym, qid);
    __syncthreads();
    const uint4 *smeta4 = reinterpret_cast<const uint4 *>(smeta);
    const uint4 *hmeta4 = reinterpret_cast<const uint4 *>(hmeta);
    uint2 *out = entries + (uint64_t)grp * nsuper;
    uint32_t nnode = 0, work = 0;
    const uint32_t hb = blockIdx.x * hyper_per_cta, he = min(hb + hyper_per_cta, nhyper);
    for (uint32_t h = hb + warp; h < he; h += NW) {
        // the hyper-node bound, lane = query
        bool alive = false;
        if (lane < G) {
            const uint4 a = __ldg(hmeta4 + 2 * (uint64_t)h), b = __ldg(hmeta4 + 2 * (uint64_t)h + 1);
            alive = node_e8(lut8_sh + lane * W * CARD, qsym[lane][0], qsym[lane][1], a, b) <= 254u;
            nnode++;
        }
        uint32_t hm = __ballot_sync(FULL, alive);
        if (!hm) continue;
        // the super-node bounds, lane = super-node (its summary loaded once for all the queries)
        const uint32_t sn = h * HYPER + lane;
        const bool ins = sn < nsuper;
        uint4 a = make_uint4(0, 0, 0, 0), b = a;
        if (ins) {
            a = __ldg(smeta4 + 2 * (uint64_t)sn);
            b = __ldg(smeta4 + 2 * (uint64_t)sn + 1);
        }
        uint32_t m = 0;  // the queries that keep this lane's super-node
#pragma unroll 1
        for (; hm; hm &= hm - 1) {
            const uint32_t g = __ffs(hm) - 1;
            const bool ok = ins && node_e8(lut8_sh + g * W * CARD, qsym[g][0], qsym[g][1], a, b) <= 254u;
            nnode += ins ? 1u : 0u;
            m |= (ok ? 1u : 0u) << g;
            if (qkept) {  // (uniform) the slot's kept super-nodes, for fbdecide_kernel
                const uint32_t balg = __ballot_sync(FULL, ok);
                if (lane == 0 && balg && g0 + g < nq) atomicAdd(&qkept[g0 + g], (uint32_t)__popc(balg));
            }
        }
        if (count_only) continue;  // (uniform: the counting pass of R15's per-query choice writes no entries)
        const bool heavy = HEAVY == 0 ? m != 0 : (uint32_t)__popc(m) >= HEAVY;
        const uint32_t balh = __ballot_sync(FULL, heavy), ball = __ballot_sync(FULL, m != 0 && !heavy);
        if (balh | ball) {
            uint32_t off = 0;
            if (lane == 0 && balh) off = atomicAdd(&ctl[CTL_WORDS * grp + CTL_CNT], (uint32_t)__popc(balh));
            if (lane == 1 && ball) off = atomicAdd(&ctl[CTL_WORDS * grp + CTL_CNT_L], (uint32_t)__popc(ball));
            const uint32_t offh = __shfl_sync(FULL, off, 0), offl = __shfl_sync(FULL, off, 1);
            ISAX_BOUND(offh + __popc(balh) + offl + __popc(ball) <= nsuper);
            if (heavy) out[offh + __popc(balh & lt)] = make_uint2(sn, m);
            else if (m) out[nsuper - 1 - (offl + __popc(ball & lt))] = make_uint2(sn, m);
            work += __popc(m);
        }
    }
    work = __reduce_add_sync(FULL, work);
    nnode = __reduce_add_sync(FULL, nnode);
    if (lane == 0) {
        if (work) atomicAdd(&ctl[CTL_WORDS * grp + CTL_WORK], work);
        if (nnode) {
            atomicAdd(scan_bytes_dev, 32ull * nnode);
            atomicAdd(scan_bytes_dev + 1, 16ull * nnode);
        }
    }
}

template <int G>
__global__ void __launch_bounds__(LF_THREADS, LF_CTAS) itemscan_kernel(
    const uint4 *__restrict__ sax, const uint8_t *__restrict__ cmeta, const uint8_t *__restrict__ lmeta, uint32_t N,
    uint32_t nleaf, uint32_t nsuper, const float *__restrict__ lut_all, const uint8_t *__restrict__ lut8_all,
    const uint4 *__restrict__ qconst_all, const uint8_t *__restrict__ qsax_all, const uint32_t *__restrict__ qmap,
    uint32_t nq, const uint2 *__restrict__ entries, uint32_t *__restrict__ ctl, uint32_t *__restrict__ cand,
    uint16_t *__restrict__ candq, uint32_t *__restrict__ cand_cnt, uint32_t cap, uint32_t *__restrict__ hist,
    uint32_t *__restrict__ leaves_alive, unsigned long long *__restrict__ scan_bytes_dev) {
    // shared: [G][16][256] u8 tables (256-aligned by hand) | per-warp scratch | per-warp candidate staging | per-warp word ring
    extern __shared__ __align__(16) uint8_t smem_dyn[];
    const uint32_t raw8 = (uint32_t)__cvta_generic_to_shared(smem_dyn);
    const uint32_t lut8_sh = (raw8 + 255u) & ~255u;
    uint8_t *lut8 = smem_dyn + (lut8_sh - raw8);
    constexpr uint32_t NW = LF_THREADS / 32;
    constexpr uint32_t WSC_ALL = (NW * WSC + 15u) & ~15u;
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t wsc_sh = lut8_sh + G * W * CARD + warp * WSC;  // this warp's scratch
    const uint32_t la_sh = wsc_sh, cl0_sh = wsc_sh + 32, iq_sh = wsc_sh + 32 + 2 * CLIST;
    uint2 *wbuf = reinterpret_cast<uint2 *>(lut8 + G * W * CARD + WSC_ALL) + warp * WB;
    const uint32_t ring = lut8_sh + G * W * CARD + WSC_ALL + NW * WB * 8 + warp * 1024 + lane * 16;  // two slots of 32 words
    uint32_t wcnt = 0;
    __shared__ QConst qc[G];
    __shared__ uint4 qsym[G][2];  // the query's 16 symbols as 8 u16x2 pairs
    __shared__ uint32_t qid[G], alive_cnt[G], s_ovf[G];
    __shared__ float qsc[G];  // 254 / T rounded down (the u8 table scale)
    __shared__ uint32_t shist[G][HIST_BINS];
    __shared__ uint32_t s_grp;
    constexpr uint32_t FULL = 0xffffffffu;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t ngroups = (nq + G - 1) / G;
    const uint4 *meta4 = reinterpret_cast<const uint4 *>(lmeta);
    const uint4 *cmeta4 = reinterpret_cast<const uint4 *>(cmeta);
    // stats: leaf tests of this thread (32 B summary, 16 lookups each); cell tests and alive cells of
    // this warp's items (each lane counts the same)
    uint32_t nnode = 0, ncellt = 0, nmembt = 0;
    // the CTA's first group: the groups share the CTAs in proportion to their work estimates
    if (t == 0) {
        unsigned long long tot = 0;
        for (uint32_t g = 0; g < ngroups; g++) tot += ctl[CTL_WORDS * g + CTL_WORK];
        const unsigned long long mine = tot * blockIdx.x / gridDim.x;
        unsigned long long acc = 0;
        uint32_t pick = 0;
        for (uint32_t g = 0; g < ngroups; g++) {
            acc += ctl[CTL_WORDS * g + CTL_WORK];
            pick = g;
            if (mine < acc) break;
        }
        s_grp = pick;
    }
    __syncthreads();
    uint32_t grp = s_grp;
    for (uint32_t visited = 0; visited < ngroups; visited++, grp = grp + 1 == ngroups ? 0 : grp + 1) {
        const uint32_t nheavy = ctl[CTL_WORDS * grp + CTL_CNT];
        const uint32_t nent = nheavy + ctl[CTL_WORDS * grp + CTL_CNT_L];
        const uint32_t g0 = grp * G;
        // one thread decides whether the group still has entries (the cursor moves under our feet);
        // the barrier also ends the previous group's flush before its tables are overwritten
        __syncthreads();
        if (t == 0) s_grp = ctl[CTL_WORDS * grp + CTL_CUR] < nent ? 1u : 0u;
        __syncthreads();
        if (!s_grp) continue;
        load_group<G, LF_THREADS>(g0, nq, qmap, qsax_all, lut8_all, lut8, qsym, qid);
        for (uint32_t e = t; e < G * HIST_BINS; e += LF_THREADS) shist[e / HIST_BINS][e % HIST_BINS] = 0;
        if (t < G) {
            const bool valid = g0 + t < nq;
            const uint32_t slot = valid ? g0 + t : g0;
            alive_cnt[t] = 0;
            s_ovf[t] = 0;
            const uint4 k = qconst_all[2 * slot], k2 = qconst_all[2 * slot + 1];
            qc[t] = valid ? QConst{__uint_as_float(k.x), __uint_as_float(k.y), k.z, k.w, k2.x, k2.y, 0u, 0u}
                          : QConst{0.f, -1.f, 0u, 0u, 0u, 0u, 0u, 0u};
            qsc[t] = valid && __uint_as_float(k.y) >= 0.f ? __fdiv_rd(254.0f, __uint_as_float(k.y)) : 0.f;  // as scanprep
        }
        __syncthreads();
        const uint2 *ent = entries + (uint64_t)grp * nsuper;
        uint32_t *cursor = &ctl[CTL_WORDS * grp + CTL_CUR];
        // ---- this warp's entries
        auto claim = [&]() -> uint2 {  // the next entry of the group (x = 0xffffffff when none is left)
            uint32_t e = 0;
            if (lane == 0) e = atomicAdd(cursor, 1u);
            e = __shfl_sync(FULL, e, 0);
            if (e >= nent) return make_uint2(0xffffffffu, 0u);
            const uint2 en = __ldg(ent + (e < nheavy ? e : nsuper - 1 - (e - nheavy)));
            const uint32_t leaf = en.x * SUPER + 4 * lane;  // its leaf summaries (32 x 32 B = eight lines) into L2
            if (lane < 8 && leaf < nleaf) prefetch_l2(meta4 + 2 * (uint64_t)leaf);
            return en;
        };
        uint32_t iq_head = 0, iq_tail = 0;  // the item ring (warp-uniform): (super-node << 4 | query, alive-leaf mask)
        // A2 of an entry: one node bound per query of its mask, lane = leaf
        auto stage_a2 = [&](uint2 en) {
            const uint32_t leaf = en.x * SUPER + lane;
            const bool inr = leaf < nleaf;
            uint4 mn4 = make_uint4(0, 0, 0, 0), mx4 = mn4;
            if (inr) {
                mn4 = __ldg(meta4 + 2 * (uint64_t)leaf);
                mx4 = __ldg(meta4 + 2 * (uint64_t)leaf + 1);
            }
            bool any_ok = false;
            uint32_t mnu[8], mxu[8];  // unpacked once for all the queries of the mask
            unpack_u16x2(mn4, mnu);
            unpack_u16x2(mx4, mxu);
#pragma unroll 1
            for (uint32_t mm = en.y; mm; mm &= mm - 1) {
                const uint32_t g = __ffs(mm) - 1;
                const bool ok = inr && node_e8_unpacked(lut8_sh + g * W * CARD, qsym[g][0], qsym[g][1], mnu, mxu) <= 254u;
                nnode += inr ? 1u : 0u;
                any_ok |= ok;
                const uint32_t bal = __ballot_sync(FULL, ok);
                if (bal) {
                    if (lane == 0) {
                        st_sh_v2a(iq_sh + (iq_tail & (IQ - 1)) * 8, (en.x << 4) | g, bal);
                        atomicAdd(&alive_cnt[g], (uint32_t)__popc(bal));  // (leaf, query) pairs that survived (stats)
                    }
                    iq_tail++;
                }
            }
            // the four cell summaries of a leaf some query kept: one 128-byte line
            if (any_ok) prefetch_l2(cmeta4 + 2 * ((uint64_t)leaf * CPL));
            __syncwarp();
        };
        // A3 of the ring's next item: lane = cell (idx & 3) of the (idx >> 2)-th alive leaf, 32 cells
        // per iteration; the alive cells go to the list at cl_sh (padded with eight copies of its
        // first entry, so that B reads and stages one iteration ahead without a bounds test).
        // Returns (item, alive cells), alive cells = 0 when none.
        auto stage_a3 = [&](uint32_t cl_sh) -> uint2 {
            const uint2 it = ld_sh_v2a(iq_sh + (iq_head & (IQ - 1)) * 8);
            iq_head++;
            const uint32_t am = it.y, sn = it.x >> 4, g = it.x & 15u;
            const uint32_t ub = lut8_sh + g * W * CARD;
            if ((am >> lane) & 1u) st_sh_u8a(la_sh + __popc(am & lt), lane);
            __syncwarp();
            const uint32_t ncell = __popc(am) * CPL;
            const uint4 qa = qsym[g][0], qb = qsym[g][1];
            const uint4 *cm0 = cmeta4 + 2 * ((uint64_t)sn * CPS);
            uint32_t m = 0;
#pragma unroll 1
            for (uint32_t j = 0; j < ncell; j += 32) {
                const uint32_t idx = j + lane;
                const bool have = idx < ncell;
                const uint32_t cell = ld_sh_u8(la_sh + (have ? idx >> 2 : 0u)) * CPL + (idx & 3u);  // in the super-node
                bool ok = false;
                if (have) {
                    const uint4 a = __ldg(cm0 + 2 * cell), b = __ldg(cm0 + 2 * cell + 1);
                    ok = node_e8(ub, qa, qb, a, b) <= 254u;
                }
                const uint32_t bal = __ballot_sync(FULL, ok);
                if (ok) {
                    st_sh_u8a(cl_sh + m + __popc(bal & lt), cell);
                    prefetch_l2(sax + (uint64_t)sn * SUPER_SIZE + cell * CELL);  // the cell's 8 words: one line
                }
                m += __popc(bal);
            }
            ncellt += ncell;
            __syncwarp();
            if (m) {
                // (B stages the cells of iteration i + 4 for i up to 4 floor((m - 1) / 4): list indices
                // up to m + 6, so seven copies are needed; a stale byte there would be a cell index
                // outside the super-node, and for the last super-nodes outside the array)
                if (lane < 8) st_sh_u8a(cl_sh + m + lane, ld_sh_u8(cl_sh));
                nmembt += m;
            }
            return make_uint2(it.x, m);
        };
        // The staged members of this warp (they passed the u8 test), one per lane: the keep rule, the
        // histogram and the append to the query's global list. The rule is the flat scan's, lo <
        // LB^2 <= T on the exact fp32 bound. A u8 sum <= E_SURE already implies LB^2 <= T (R11b), and
        // in the first band (lo < 0) lo < LB^2 always holds: there, members with a u8 sum in
        // (E_SURE, 254] are kept marked B_UNCHECKED and get the exact rule in candcheck_kernel; in
        // later bands every member gets it here (its word is read again: a rare path). A first-band
        // member's histogram bin comes from its u8 sum, never above its exact bin (band shrinking,
        // R10, stays an upper bound on the count). The entries of one query get one global atomic
        // (match_any groups the lanes); once a query's list has passed its capacity its flag stops
        // this CTA's appends (the list is dropped for the round anyway, R10).
        auto flush_staged = [&]() {
            __syncwarp();
            for (uint32_t i0 = 0; i0 < wcnt; i0 += 32) {
                const bool have = i0 + lane < wcnt;
                const uint2 en = have ? wbuf[i0 + lane] : make_uint2(0u, 0u);
                const uint32_t g = (en.y >> 16) & 15u, e8 = en.y & 0xFFu, e8hi = (en.y >> 8) & 0xFFu, pos = en.x;
                const QConst kq = qc[g];
                const bool band0 = kq.lo < 0.f;
                float lb = 0.f;
                if (have && !band0) lb = word_lb(lut_all + (uint64_t)qid[g] * W * CARD, __ldg(sax + pos));
                const bool keep = have && (band0 || (lb > kq.lo && lb <= kq.T)) && pos_ok(kq, pos) && pos < N;
                // the candidate's u8 bound b <= LB^2 * sc (for the refine), or B_UNCHECKED
                uint32_t b = e8 <= E_SURE ? e8 : B_UNCHECKED;
                if (!band0) {
                    const float y = __fmul_rd(lb, qsc[g]);
                    b = lb > 0.f ? (y >= 254.f ? 254u : (uint32_t)y) : 0u;
                }
                if (keep) atomicAdd(&shist[g][band0 ? min(e8 * HIST_BINS / 254u, HIST_BINS - 1) : hist_bin(lb, kq.lo, kq.T)], 1u);
                const uint32_t peers = __match_any_sync(FULL, keep ? g : 0xFFFFu);
                if (keep) {
                    const uint32_t leader = __ffs(peers) - 1;
                    const uint32_t q = qid[g];
                    uint32_t base = 0xffffffffu;
                    if (lane == leader && !s_ovf[g]) {
                        const uint32_t c = __popc(peers);
                        base = atomicAdd(&cand_cnt[q], c);
                        if (base + c > cap) s_ovf[g] = 1u;
                    }
                    base = __shfl_sync(peers, base, leader);
                    const uint32_t k = base + __popc(peers & lt);
                    ISAX_BOUND(pos < N);
                    if (base != 0xffffffffu && k < cap) {
                        cand[(uint64_t)q * cap + k] = pos;
                        candq[(uint64_t)q * cap + k] = (uint16_t)(b | (e8hi << 8));
                    }
                }
            }
            __syncwarp();
            wcnt = 0;
        };
        // B of an item: quarter warp = alive cell, lane = member. Each lane stages its own word of
        // the next iteration's cell (cp.async into the warp's other slot) before this one's lookups.
        auto stage_b = [&](uint32_t item, uint32_t m, uint32_t cl_sh) {
            const uint32_t sn = item >> 4, g = item & 15u;
            const uint32_t ub = lut8_sh + g * W * CARD;
            const char *wbase = reinterpret_cast<const char *>(sax + (lane & 7u));
            const uint32_t cell0 = sn * CPS;
            const uint32_t clp = cl_sh + (lane >> 3);
            const int lim = (int)m - (int)(lane >> 3);  // this quarter has a cell while i < lim
            cp_async16_sh(ring, wbase + (uint64_t)(cell0 + ld_sh_u8(clp)) * (CELL * 16));
            cp_async_commit();
            uint32_t slot = 0;
#pragma unroll 1
            for (uint32_t i = 0; i < m; i += 4) {
                cp_async16_sh(ring + (slot ^ 512u), wbase + (uint64_t)(cell0 + ld_sh_u8(clp + i + 4)) * (CELL * 16));
                cp_async_commit();
                cp_async_wait<1>();
                const uint4 wv = ld_sh_v4a(ring + slot);
                slot ^= 512u;
                uint32_t e8hi;
                const uint32_t e8 = word_e8(ub, wv, e8hi);
                const bool maybe = (int)i < lim && e8 <= 254u;
                // Members that pass the u8 test are only staged here: (position, query | u8 sums) into
                // the warp's buffer. The keep rule runs when the buffer is emptied, one staged member
                // per lane (flush_staged), instead of once per passing warp iteration for one or two
                // live lanes.
                const uint32_t bal = __ballot_sync(FULL, maybe);
                if (!bal) continue;
                if (maybe)
                    wbuf[wcnt + __popc(bal & lt)] =
                        make_uint2((cell0 + ld_sh_u8(clp + i)) * CELL + (lane & 7u), (g << 16) | (e8hi << 8) | e8);
                wcnt += __popc(bal);
                if (wcnt > WB - 32) flush_staged();
            }
            cp_async_wait<0>();  // the trailing copy (a repeat of the first cell)
        };
        uint2 en_n = claim();  // the next entry (claimed an entry ahead)
        uint2 prev = make_uint2(0u, 0u);  // the item B runs next (y = its alive cells; its list is list `buf`)
        uint32_t buf = 0;
        for (;;) {
            // refill the ring when it holds at most one item
            while (iq_tail - iq_head <= 1u && en_n.x != 0xffffffffu) {
                const uint2 en = en_n;
                en_n = claim();
                stage_a2(en);
            }
            if (iq_tail == iq_head) break;
            const uint2 it = stage_a3(cl0_sh + (buf ^ 1u) * CLIST);
            if (prev.y) stage_b(prev.x, prev.y, cl0_sh + buf * CLIST);
            if (it.y) {
                prev = it;
                buf ^= 1u;
            } else if (prev.y) {
                prev.y = 0;  // B ran; the list `buf` is free again, and the new one held nothing
            }
        }
        if (prev.y) stage_b(prev.x, prev.y, cl0_sh + buf * CLIST);
        if (wcnt) flush_staged();  // (warp-uniform)
        // the group's histograms and surviving-leaf counts into global memory
        __syncthreads();
        if (t < G && alive_cnt[t] && g0 + t < nq) atomicAdd(&leaves_alive[qid[t]], alive_cnt[t]);
        for (uint32_t e = t; e < G * HIST_BINS; e += LF_THREADS) {
            const uint32_t g = e / HIST_BINS, b = e % HIST_BINS;
            if (g0 + g < nq && shist[g][b]) atomicAdd(&hist[qid[g] * HIST_BINS + b], shist[g][b]);
        }
    }
    // stats: bytes of summaries and words read, and the lookups made (16 per test; an alive cell is
    // CELL member tests of 16 B and 16 lookups each)
    const unsigned long long nodes = (unsigned long long)__reduce_add_sync(FULL, nnode) + ncellt;
    const unsigned long long membs = (unsigned long long)nmembt * CELL;
    if (lane == 0 && nodes) {
        atomicAdd(scan_bytes_dev, nodes * 32ull + membs * 16ull);
        atomicAdd(scan_bytes_dev + 1, 16ull * (nodes + membs));
    }
}

#ifndef ISAX_TASKS_PER_SM
#define ISAX_TASKS_PER_SM 16
#endif

template <int G>
static void launch_leaf(const isax_index *ix, uint32_t nq, const uint32_t *qmap, const Band *band, float onepd, bool select,
                        cudaStream_t s) {
    constexpr uint32_t NW = LF_THREADS / 32;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t groups = (nq + G - 1) / G;
    const uint32_t nleaf = (uint32_t)((ix->N + LEAF - 1) / LEAF);
    const QueryScratch &qs = ix->qs;
#if ISAX_SCAN_V1
    const size_t smem = (size_t)G * (W * CARD + CW) + 256 + CHUNK * 4 + (size_t)NW * PD * LEAF * sizeof(uint4) +
                        (size_t)NW * WB * sizeof(uint2) + (size_t)NW * SV * 20;
    // per launch (the attribute is per device; a failure surfaces as the launch's error)
    cudaFuncSetAttribute(leafscan_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // chunk: as large as possible (fewer phase barriers) while leaving >= 16 tasks per SM for
    // balance; a power of two >= 512, so a multiple of SUPER
    uint32_t chunk = CHUNK;
    while (chunk > 512 && (uint64_t)groups * ((nleaf + chunk - 1) / chunk) < (uint64_t)ISAX_TASKS_PER_SM * sms) chunk >>= 1;
    const uint64_t tasks = (uint64_t)groups * ((nleaf + chunk - 1) / chunk);
    const unsigned grid = (unsigned)std::max<uint64_t>(1, umin64(tasks, (uint64_t)sms * LF_CTAS));
    // one task per grab: runs of 4-8 consecutive chunks per CTA (fewer table reloads with many
    // groups) measured 30-100% slower: the CTAs then stream through scattered parts of the arrays
    leafscan_kernel<G><<<grid, LF_THREADS, smem, s>>>(
        reinterpret_cast<const uint4 *>(ix->sax), ix->lmeta, ix->smeta, ix->hmeta, (uint32_t)ix->N, qs.lut, qs.lut8, qs.lut8c,
        qs.qconst, qs.qsax, qmap, nq, nleaf, chunk, qs.cand, qs.candq, qs.cand_cnt, qs.cand_cap, qs.cand_hist, qs.counters_leaf,
        qs.scan_bytes_dev, qs.task_ctr, 1u);
#else
    const uint32_t nsuper = (nleaf + SUPER - 1) / SUPER, nhyper = (nsuper + HYPER - 1) / HYPER;
    // node scan: a CTA per (block of hyper-nodes, group); blocks sized for about three CTAs per SM in all
    const size_t smem_n = (size_t)G * W * CARD + 256;
    cudaFuncSetAttribute(nodescan_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_n);
    const uint32_t want = std::max(1u, (uint32_t)sms * 3u / groups);
    const uint32_t hpc = std::max(8u, (nhyper + want - 1) / want);
    // R15 per query: a counting pass of the node scan under the whole window threshold, then only the
    // queries that kept many super-nodes get the first band (fbdecide_kernel), then the node scan proper
    if (select) {
        nodescan_kernel<G><<<dim3((nhyper + hpc - 1) / hpc, groups), NS_THREADS, smem_n, s>>>(
            ix->smeta, ix->hmeta, nsuper, nhyper, qs.lut8, qs.qsax, qmap, nq, hpc, qs.scan_entries, qs.scan_ctl, qs.scan_bytes_dev,
            qs.qkept, true);
// (a query is costly when it keeps more than 1/16 of the super-nodes: config 5 1.03M q/s with 1/256,
// 1.06M with 1/64, 1.08M with 1/16, 1.03M with 1/4)
#ifndef ISAX_FB_HEAVY_DIV
#define ISAX_FB_HEAVY_DIV 16
#endif
        fbdecide_kernel<<<nq, 256, 0, s>>>(qs.lut, qmap, band, qs.bsf, onepd, qs.qkept, std::max(32u, nsuper / ISAX_FB_HEAVY_DIV), qs.lut8,
                                           qs.qconst, qs.qscale, qs.qT, qs.bsf_scan);
    }
    nodescan_kernel<G><<<dim3((nhyper + hpc - 1) / hpc, groups), NS_THREADS, smem_n, s>>>(
        ix->smeta, ix->hmeta, nsuper, nhyper, qs.lut8, qs.qsax, qmap, nq, hpc, qs.scan_entries, qs.scan_ctl, qs.scan_bytes_dev,
        nullptr, false);
    // item scan: persistent CTAs, no more than the entries can occupy
    const size_t smem = (size_t)G * W * CARD + 256 + ((NW * WSC + 15u) & ~15u) + (size_t)NW * WB * sizeof(uint2) +
                        (size_t)NW * 1024;
    cudaFuncSetAttribute(itemscan_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const unsigned grid = (unsigned)std::max<uint64_t>(
        1, umin64(((uint64_t)nsuper * groups + NW - 1) / NW, (uint64_t)sms * LF_CTAS));
    itemscan_kernel<G><<<grid, LF_THREADS, smem, s>>>(
        reinterpret_cast<const uint4 *>(ix->sax), ix->cmeta, ix->lmeta, (uint32_t)ix->N, nleaf, nsuper, qs.lut, qs.lut8,
        qs.qconst, qs.qsax, qmap, nq, qs.scan_entries, qs.scan_ctl, qs.cand, qs.candq, qs.cand_cnt, qs.cand_cap, qs.cand_hist,
        qs.counters_leaf, qs.scan_bytes_dev);
#endif
}

uint64_t launch_lbscan(const isax_index *ix, uint32_t nq, uint32_t B, const uint32_t *qmap, const Band *band,
                       float delta, bool select_first_band, cudaStream_t s) {
    if (!nq) return 0;
    const float onepd = 1.0f + delta;
    const QueryScratch &qs = ix->qs;
    // (the per-query choice needs the node scan's counts: the default scan only)
    const bool select = select_first_band && !(ix->opts.flags & ISAX_FLAG_FLAT_SCAN) && !ISAX_SCAN_V1;
    scanprep_kernel<<<nq, 256, 0, s>>>(qs.lut, qmap, band, qs.bsf, qs.win, onepd, qs.lut8, qs.lut8c, qs.qconst, qs.qscale, qs.qT, qs.bsf_scan,
                                      B, qs.cand_cnt, qs.cand_cnt2, qs.cnt_hi, qs.cnt_f, qs.cand_hist, qs.task_ctr, qs.scan_ctl,
                                      4u * qs.scan_groups, qs.qkept, select);
    if (ix->opts.flags & ISAX_FLAG_FLAT_SCAN) {  // ParIS flat scan, kept for A/B measurement
        const uint32_t G = nq >= 4 ? 4 : nq;
        if (G == 4) launch_g<4>(ix, nq, qmap, band, onepd, s);
        else if (G == 3) launch_g<3>(ix, nq, qmap, band, onepd, s);
        else if (G == 2) launch_g<2>(ix, nq, qmap, band, onepd, s);
        else launch_g<1>(ix, nq, qmap, band, onepd, s);
        return 16ull * ix->N * ((nq + G - 1) / G);  // words read
    }
#ifndef ISAX_GMAX
#define ISAX_GMAX 16  // queries per scan group (their u8 tables share a CTA's shared memory)
#endif
    const uint32_t G = nq >= 16 && ISAX_GMAX >= 16 ? 16 : nq >= 8 && ISAX_GMAX >= 8 ? 8 : nq >= 4 ? 4 : nq >= 2 ? 2 : 1;
    if (G == 16) launch_leaf<16>(ix, nq, qmap, band, onepd, select, s);
    else if (G == 8) launch_leaf<8>(ix, nq, qmap, band, onepd, select, s);
    else if (G == 4) launch_leaf<4>(ix, nq, qmap, band, onepd, select, s);
    else if (G == 2) launch_leaf<2>(ix, nq, qmap, band, onepd, select, s);
    else launch_leaf<1>(ix, nq, qmap, band, onepd, select, s);
    return 0;  // the leaf scan counts the node summaries and words it reads on the device
}

// ------------------------------------------------------------------------------------ candcheck
// The exact fp32 rule (LB^2 <= T, the flat scan's) for the candidates the leaf scan kept on their
// u8 sum alone (candq == B_UNCHECKED), many at a time: a CTA takes a slice of the flat candidate
// index (all queries' lists back to back), loads the fp32 LUT of each query it meets into shared
// memory, and each thread tests one candidate (its word from the sorted SAX array, 16 shared
// lookups summed left to right). Every list is compacted into cand2 (order is immaterial, R9);
// the kept ones' u8 bound becomes floor(LB^2 * sc).
constexpr int CK_THREADS = 256;
#ifndef ISAX_BSPLIT
#define ISAX_BSPLIT 140
#endif
constexpr uint32_t B_SPLIT = ISAX_BSPLIT;  // second refine pass: b > B_SPLIT, i.e. LB^2 above about 0.55 T
#ifndef ISAX_SPLIT_MIN
#define ISAX_SPLIT_MIN 4096
#endif
constexpr uint32_t SPLIT_MIN = ISAX_SPLIT_MIN;  // ... for queries with more candidates than this
constexpr uint32_t SPLIT_TARGET = 65536;  // first-pass size a lowered split aims at

// three CTAs per SM (at most 80 registers; 92 allowed only two): the kernel is latency-bound on
// its word and table loads, so the extra warps pay (cfg3 0.074 -> 0.057 ms)
#ifndef ISAX_CK_MINB
#define ISAX_CK_MINB 3
#endif
__global__ void __launch_bounds__(CK_THREADS, ISAX_CK_MINB) candcheck_kernel(
    const uint32_t *__restrict__ cand, const uint16_t *__restrict__ candq, const uint32_t *__restrict__ cand_cnt,
    uint32_t Q, uint32_t cap, const uint4 *__restrict__ sax, const float *__restrict__ lut_all,
    const float *__restrict__ qT, const float *__restrict__ qscale, uint32_t *__restrict__ cand2,
    uint16_t *__restrict__ candq2, uint32_t *__restrict__ cand_cnt2, uint32_t *__restrict__ cnt_hi,
    const uint32_t *__restrict__ hist) {
    constexpr int U = 8;  // candidates per thread per iteration, all loads in flight together
    __shared__ uint32_t pre[1025];
    __shared__ __align__(16) float slut[W * CARD];
    constexpr uint32_t FULL = 0xffffffffu;
    const uint32_t t = threadIdx.x, lane = t & 31;
    const uint32_t lt = (1u << lane) - 1u;
    cand_prefix<CK_THREADS>(cand_cnt, Q, cap, pre);
    const uint32_t total = pre[Q];
    // one contiguous slice per CTA; the LUT of the slice's first query goes to shared memory
    // (lanes of a later query read the global LUT)
    const uint32_t per = (total + gridDim.x - 1) / gridDim.x;
    const uint32_t f0 = min(blockIdx.x * per, total), f1 = min(f0 + per, total);
    if (f0 >= f1) return;
    uint32_t q0;
    {
        uint32_t lo = 0, hi = Q;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (pre[mid] <= f0) lo = mid;
            else hi = mid;
        }
        q0 = lo;
    }
    // the split of q0's list between the two refine passes: B_SPLIT, lowered so that the first
    // pass holds about SPLIT_TARGET candidates when the scan's histogram of LB^2 / T (R10; bins
    // of width T / 64 = 254 / 64 u8 units) says the list is much longer
    __shared__ uint32_t s_b1;
    if (t < 32) {
        const uint32_t c = hist[q0 * HIST_BINS + 2 * t] + hist[q0 * HIST_BINS + 2 * t + 1];
        uint32_t inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(FULL, inc, o);
            if (t >= (uint32_t)o) inc += u;
        }
        const uint32_t over = __ballot_sync(FULL, inc >= SPLIT_TARGET);
        uint32_t b1 = B_SPLIT;
        if (over) b1 = min(B_SPLIT, (2u * (__ffs(over) - 1) + 2u) * 254u / HIST_BINS);
        if (t == 0) s_b1 = b1;
    }
    {
        const float4 *src = reinterpret_cast<const float4 *>(lut_all + (uint64_t)q0 * W * CARD);
        float4 v[W * CARD / 4 / CK_THREADS];
#pragma unroll
        for (int k = 0; k < W * CARD / 4 / CK_THREADS; k++) v[k] = __ldg(src + k * CK_THREADS + t);
#pragma unroll
        for (int k = 0; k < W * CARD / 4 / CK_THREADS; k++) reinterpret_cast<float4 *>(slut)[k * CK_THREADS + t] = v[k];
    }
    __syncthreads();
    const uint32_t b1 = s_b1;
    uint32_t q = q0;  // a thread's query only moves forward
    for (uint32_t fb = f0; fb < f1; fb += U * CK_THREADS) {
        uint32_t qk[U], pos[U], b[U], b2[U];
        bool valid[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t f = fb + u * CK_THREADS + t;
            valid[u] = f < f1;
            if (valid[u])
                while (pre[q + 1] <= f) q++;
            qk[u] = q;
            const uint64_t k = (uint64_t)q * cap + (f - pre[q]);
            pos[u] = valid[u] ? cand[k] : 0u;
            const uint32_t bq = valid[u] ? candq[k] : 0u;
            b[u] = bq & 0xFFu;
            b2[u] = bq >> 8;  // the second half's bound (R16), passed through
        }
        uint4 wv[U];
#pragma unroll
        for (int u = 0; u < U; u++) wv[u] = valid[u] && b[u] == B_UNCHECKED ? __ldg(sax + pos[u]) : make_uint4(0, 0, 0, 0);
        bool keep[U];
        bool one_q = true;  // this lane's U candidates share one query
#pragma unroll
        for (int u = 0; u < U; u++) {
            keep[u] = valid[u];
            one_q &= !valid[u] || qk[u] == qk[0];
            if (valid[u] && b[u] == B_UNCHECKED) {
                const float *L = qk[u] == q0 ? slut : lut_all + (uint64_t)qk[u] * W * CARD;
                const float lb = word_lb(L, wv[u]);
                keep[u] = lb <= qT[qk[u]];  // first band: lo < 0 <= LB^2 always
                const float y = __fmul_rd(lb, qscale[qk[u]]);
                b[u] = lb > 0.f ? (y >= 254.f ? 254u : (uint32_t)y) : 0u;
            }
        }
        // Append to the query's lists in cand2: the first refine pass's from the front, and for a
        // query with more than SPLIT_MIN candidates the ones with b > B_SPLIT (LB^2 above about
        // 0.55 T) from the back, for the second pass (refine.cu). One global atomic per list per
        // warp when the whole warp's candidates share a query (the common case), else one per
        // (query, list, u) peer group.
        bool hi[U];
#pragma unroll
        for (int u = 0; u < U; u++)
            hi[u] = keep[u] && b[u] > (qk[u] == q0 ? b1 : B_SPLIT) && pre[qk[u] + 1] - pre[qk[u]] > SPLIT_MIN;
        auto put = [&](uint32_t qq, uint32_t idx, bool h, uint32_t p, uint32_t bb) {
            ISAX_BOUND(idx < cap && qq < Q);
            const uint64_t k2 = (uint64_t)qq * cap + (h ? cap - 1 - idx : idx);
            cand2[k2] = p;
            candq2[k2] = (uint16_t)bb;
        };
        const uint32_t q_lane = qk[0];
        const uint32_t q_w = __shfl_sync(FULL, q_lane, 0);  // (every lane shuffles: no short circuit)
        if (__all_sync(FULL, one_q && q_lane == q_w)) {
            uint32_t bl[U], bh[U], cl = 0, ch = 0;
#pragma unroll
            for (int u = 0; u < U; u++) {
                bl[u] = __ballot_sync(FULL, keep[u] && !hi[u]);
                bh[u] = __ballot_sync(FULL, hi[u]);
                cl += __popc(bl[u]);
                ch += __popc(bh[u]);
            }
            uint32_t base = 0;
            if (lane == 0 && cl) base = atomicAdd(&cand_cnt2[q_lane], cl);
            if (lane == 1 && ch) base = atomicAdd(&cnt_hi[q_lane], ch);
            uint32_t basel = __shfl_sync(FULL, base, 0), baseh = __shfl_sync(FULL, base, 1);
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (keep[u] && !hi[u]) put(q_lane, basel + __popc(bl[u] & lt), false, pos[u], b[u] | (b2[u] << 8));
                if (hi[u]) put(q_lane, baseh + __popc(bh[u] & lt), true, pos[u], b[u] | (b2[u] << 8));
                basel += __popc(bl[u]);
                baseh += __popc(bh[u]);
            }
        } else {
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t peers = __match_any_sync(FULL, keep[u] ? 2 * qk[u] + (hi[u] ? 1u : 0u) : 0xffffffffu);
                if (keep[u]) {
                    const uint32_t leader = __ffs(peers) - 1;
                    uint32_t base = 0;
                    if (lane == leader) base = atomicAdd(hi[u] ? &cnt_hi[qk[u]] : &cand_cnt2[qk[u]], (uint32_t)__popc(peers));
                    base = __shfl_sync(peers, base, leader);
                    put(qk[u], base + __popc(peers & lt), hi[u], pos[u], b[u] | (b2[u] << 8));
                }
            }
        }
    }
}

void launch_candcheck(const isax_index *ix, uint32_t Q, cudaStream_t s) {
    const QueryScratch &qs = ix->qs;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // one wave (three CTAs fit an SM): every CTA pays the prefix over the lists and a 16 KB table once
    // (eight CTAs per SM: cfg3 0.068 -> 0.055 ms with three, cfg5 0.033 -> 0.027)
#ifndef ISAX_CK_GRID
#define ISAX_CK_GRID 3
#endif
    const unsigned grid = (unsigned)sms * ISAX_CK_GRID;  // the total is only known on the device
    candcheck_kernel<<<grid, CK_THREADS, 0, s>>>(qs.cand, qs.candq, qs.cand_cnt, Q, qs.cand_cap,
                                                 reinterpret_cast<const uint4 *>(ix->sax), qs.lut, qs.qT, qs.qscale,
                                                 qs.cand2, qs.candq2, qs.cand_cnt2, qs.cnt_hi, qs.cand_hist);
}

// ------------------------------------------------------------------------------------ leaf meta
// Build: per box of `box` consecutive sorted positions (a leaf of LEAF, or a kd cell of CELL rows),
// the per-segment min and max symbol of its members below N, 32 bytes. A box with no member gets
// min 255 / max 0.
__global__ void box_meta_kernel(const uint4 *__restrict__ sax, uint64_t N, uint32_t box, uint64_t nbox,
                                uint8_t *__restrict__ meta) {
    for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < nbox; l += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t mn[4] = {~0u, ~0u, ~0u, ~0u}, mx[4] = {0, 0, 0, 0};
        const uint64_t p1 = umin64(N, (l + 1) * box);
        for (uint64_t p = l * box; p < p1; p++) {
            const uint4 w = __ldg(sax + p);
            const uint32_t v[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int k = 0; k < 4; k++) {
                mn[k] = __vminu4(mn[k], v[k]);
                mx[k] = __vmaxu4(mx[k], v[k]);
            }
        }
        uint4 *o = reinterpret_cast<uint4 *>(meta + l * 32);
        o[0] = make_uint4(mn[0], mn[1], mn[2], mn[3]);
        o[1] = make_uint4(mx[0], mx[1], mx[2], mx[3]);
    }
}

// Build: per parent node of `factor` children, the per-segment min / max over its children's
// summaries (super-nodes over leaves, hyper-nodes over super-nodes).
__global__ void parent_meta_kernel(const uint4 *__restrict__ child, uint64_t nchild, uint32_t factor,
                                   uint4 *__restrict__ parent) {
    const uint64_t np = (nchild + factor - 1) / factor;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < np; j += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t mn[4] = {~0u, ~0u, ~0u, ~0u}, mx[4] = {0, 0, 0, 0};
        const uint64_t l1 = umin64(nchild, (j + 1) * factor);
        for (uint64_t l = j * factor; l < l1; l++) {
            const uint4 a = __ldg(child + 2 * l), b = __ldg(child + 2 * l + 1);
            const uint32_t va[4] = {a.x, a.y, a.z, a.w}, vb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int k = 0; k < 4; k++) {
                mn[k] = __vminu4(mn[k], va[k]);
                mx[k] = __vmaxu4(mx[k], vb[k]);
            }
        }
        parent[2 * j] = make_uint4(mn[0], mn[1], mn[2], mn[3]);
        parent[2 * j + 1] = make_uint4(mx[0], mx[1], mx[2], mx[3]);
    }
}

void launch_leaf_meta(const uint8_t *sax, uint64_t N, uint8_t *cmeta, uint8_t *lmeta, uint8_t *smeta, uint8_t *hmeta,
                      cudaStream_t s) {
    const uint64_t nleaf = (N + LEAF - 1) / LEAF;
    const uint64_t ncell = nleaf * (LEAF / KD_CELL);  // whole leaves (the SAX array is padded to them)
    auto grid = [](uint64_t n) { return (unsigned)std::max<uint64_t>(1, umin64((n + 255) / 256, 148 * 16)); };
    box_meta_kernel<<<grid(ncell), 256, 0, s>>>(reinterpret_cast<const uint4 *>(sax), N, KD_CELL, ncell, cmeta);
    box_meta_kernel<<<grid(nleaf), 256, 0, s>>>(reinterpret_cast<const uint4 *>(sax), N, LEAF, nleaf, lmeta);
    const uint64_t ns = (nleaf + SUPER - 1) / SUPER;
    parent_meta_kernel<<<grid(ns), 256, 0, s>>>(reinterpret_cast<const uint4 *>(lmeta), nleaf, SUPER,
                                                reinterpret_cast<uint4 *>(smeta));
    const uint64_t nh = (ns + HYPER - 1) / HYPER;
    parent_meta_kernel<<<grid(nh), 256, 0, s>>>(reinterpret_cast<const uint4 *>(smeta), ns, HYPER,
                                                reinterpret_cast<uint4 *>(hmeta));
}

}  // namespace isax
