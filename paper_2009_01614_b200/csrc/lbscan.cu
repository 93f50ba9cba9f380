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

struct __align__(16) QConst {  // per query slot, read with one 16-byte shared load
    float T, Tb;               // T = bsf^2 (1 + delta); Tb = T (1 + 2^-19) for the node bound
    uint32_t ws, we;           // window [ws, we): already refined, never a candidate
};

constexpr uint32_t CHUNK = 8192;  // leaves per phase-A/phase-B round of a CTA
constexpr uint32_t CBUF = 1024;   // shared candidate buffer per query slot

// append `keep` lanes' positions for query slot g: shared buffer first, global list if it is full
__device__ __forceinline__ void emit(bool keep, uint32_t pos, uint32_t g, uint32_t q, uint32_t lane, uint32_t lt,
                                     uint32_t *cbuf, uint32_t *cb_cnt, uint32_t *cand, uint32_t *cand_cnt,
                                     uint32_t cap) {
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (!bal) return;
    const uint32_t c = __popc(bal);
    uint32_t off = 0;
    if (lane == 0) off = atomicAdd(&cb_cnt[g], c);
    off = __shfl_sync(0xffffffffu, off, 0);
    const uint32_t r = __popc(bal & lt);
    if (off + c <= CBUF) {
        if (keep) cbuf[g * CBUF + off + r] = pos;
        return;
    }
    // the buffer fills up: the slots below CBUF are still written (the flush copies exactly
    // min(count, CBUF) entries), the rest go straight to the global list
    const uint32_t room = off < CBUF ? CBUF - off : 0;
    if (keep && r < room) cbuf[g * CBUF + off + r] = pos;
    uint32_t goff = 0;
    if (lane == 0) goff = atomicAdd(&cand_cnt[q], c - room);
    goff = __shfl_sync(0xffffffffu, goff, 0);
    if (keep && r >= room) {
        const uint32_t k = goff + r - room;
        if (k < cap) cand[(uint64_t)q * cap + k] = pos;
    }
}

__device__ __forceinline__ uint32_t byte_of(const uint32_t (&v)[4], int s) { return (v[s >> 2] >> (8 * (s & 3))) & 0xFFu; }

// The kernel runs two phases per chunk of CHUNK leaves:
//  A. lane = leaf: node LB^2 = sum_s LUT[s][clamp(q_s, min_s, max_s)], summed over s = 0..15
//     left to right, exactly like the per-series LB. Every term is <= the member's term and
//     fp32 addition is monotone, so node LB^2 <= member LB^2 holds exactly. Surviving leaves
//     and their query masks go to a shared worklist.
//  B. warps stream the worklist with two leaves' 1 KB of words in flight, and run the
//     per-series test for each query that kept the leaf. Candidates are buffered in shared
//     memory per query slot and flushed once per CTA (one global atomic per slot).
template <int G>
__global__ void __launch_bounds__(LF_THREADS, 1) leafscan_kernel(
    const uint4 *__restrict__ sax, const uint8_t *__restrict__ lmeta, uint32_t N, const float *__restrict__ lut_all,
    const uint8_t *__restrict__ qsax_all, const uint32_t *__restrict__ qmap, const uint32_t *__restrict__ qrange,
    uint32_t nq, uint32_t leaf_lo, uint32_t leaf_hi, uint32_t chunk, const unsigned long long *__restrict__ bsf,
    const uint32_t *__restrict__ win, float onepd, uint32_t *__restrict__ cand, uint32_t *__restrict__ cand_cnt,
    uint32_t cap, uint32_t *__restrict__ leaves_alive, unsigned long long *__restrict__ leaf_loads,
    uint32_t *__restrict__ task_ctr) {
    extern __shared__ __align__(16) float slut[];  // [G][16][256] LUTs, [G][CBUF] candidates, [CHUNK] worklist
    uint32_t *cbuf = reinterpret_cast<uint32_t *>(slut + G * W * CARD);
    uint32_t *worklist = cbuf + G * CBUF;  // (leaf offset in chunk) | (query mask << 16)
    __shared__ QConst qc[G];
    __shared__ uint4 qsym[G];
    __shared__ uint32_t r0[G], r1[G], qid[G], cb_cnt[G], alive_cnt[G], fbase[G];
    __shared__ uint32_t wl_cnt, s_task;
    __shared__ int restricted;
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    constexpr uint32_t NW = LF_THREADS / 32;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t nchunks = (leaf_hi - leaf_lo + chunk - 1) / chunk;
    const uint32_t ngroups = (nq + G - 1) / G;
    const uint32_t ntasks = nchunks * ngroups;
    const uint4 *meta4 = reinterpret_cast<const uint4 *>(lmeta);
    uint32_t loads = 0;
    uint32_t g0 = 0xffffffffu;  // first query slot of the group whose LUTs are loaded
    bool restr = false;
    // empty the shared candidate buffers of the loaded group into the global lists
    auto flush = [&]() {
        if (t < G) {
            const uint32_t c = min(cb_cnt[t], CBUF);
            fbase[t] = (c && g0 + t < nq) ? atomicAdd(&cand_cnt[qid[t]], c) : 0;
            if (alive_cnt[t] && g0 + t < nq) atomicAdd(&leaves_alive[qid[t]], alive_cnt[t]);
        }
        __syncthreads();
        for (uint32_t g = 0; g < G; g++) {
            if (g0 + g >= nq) break;
            const uint32_t c = min(cb_cnt[g], CBUF);
            for (uint32_t i = t; i < c; i += LF_THREADS) {
                const uint32_t k = fbase[g] + i;
                if (k < cap) cand[(uint64_t)qid[g] * cap + k] = cbuf[g * CBUF + i];
            }
        }
        __syncthreads();
    };
    if (t == 0) wl_cnt = 0;
    // persistent CTA: tasks (group, chunk) in group-major order from an atomic counter
    for (;;) {
        if (t == 0) s_task = atomicAdd(task_ctr, 1u);
        __syncthreads();
        const uint32_t task = s_task;
        if (task >= ntasks) break;
        const uint32_t grp = task / nchunks, ch = task % nchunks;
        if (grp * G != g0) {
            if (g0 != 0xffffffffu) flush();
            g0 = grp * G;
            for (uint32_t e = t; e < G * W * CARD; e += LF_THREADS) {
                const uint32_t g = e / (W * CARD);
                const uint32_t qi = g0 + g < nq ? qmap[g0 + g] : qmap[g0];
                slut[e] = lut_all[(uint64_t)qi * W * CARD + (e % (W * CARD))];
            }
            if (t == 0) restricted = 0;
            __syncthreads();
            if (t < G) {
                const bool valid = g0 + t < nq;
                const uint32_t qi = valid ? qmap[g0 + t] : qmap[g0];
                qid[t] = qi;
                cb_cnt[t] = 0;
                alive_cnt[t] = 0;
                qsym[t] = reinterpret_cast<const uint4 *>(qsax_all)[qi];
                const float tq = valid ? bsf_d2(bsf[qi]) * onepd : -1.0f;  // an invalid slot keeps nothing
                qc[t] = QConst{tq, tq, win[2 * qi], win[2 * qi + 1]};
                r0[t] = valid ? qrange[2 * (g0 + t)] : 0;
                r1[t] = valid ? qrange[2 * (g0 + t) + 1] : 0;
                if (valid && (r0[t] > leaf_lo * LEAF || r1[t] < min(leaf_hi * LEAF, N))) atomicOr(&restricted, 1);
            }
            __syncthreads();
            restr = restricted != 0;
        }
        {
        const uint32_t c0 = leaf_lo + ch * chunk;
        const uint32_t c1 = min(c0 + chunk, leaf_hi);
        // ---- phase A: lane = leaf; warp w takes leaves c0 + 32 w + lane, then + 32 NW, ...
        uint32_t leaf = c0 + warp * 32 + lane;
        uint4 mn_n = make_uint4(0, 0, 0, 0), mx_n = make_uint4(~0u, ~0u, ~0u, ~0u);
        if (leaf < c1) {
            mn_n = __ldg(meta4 + 2 * (uint64_t)leaf);
            mx_n = __ldg(meta4 + 2 * (uint64_t)leaf + 1);
        }
        for (; leaf - lane < c1; leaf += 32 * NW) {
            const uint32_t mn[4] = {mn_n.x, mn_n.y, mn_n.z, mn_n.w};
            const uint32_t mx[4] = {mx_n.x, mx_n.y, mx_n.z, mx_n.w};
            const uint32_t nxt = leaf + 32 * NW;
            if (nxt < c1) {
                mn_n = __ldg(meta4 + 2 * (uint64_t)nxt);
                mx_n = __ldg(meta4 + 2 * (uint64_t)nxt + 1);
            }
            uint32_t alive = 0;
#pragma unroll
            for (int g = 0; g < G; g++) {
                const uint4 q4 = qsym[g];
                const uint32_t qv[4] = {q4.x, q4.y, q4.z, q4.w};
                uint32_t cl[4];
#pragma unroll
                for (int k = 0; k < 4; k++) cl[k] = __vminu4(__vmaxu4(qv[k], mn[k]), mx[k]);
                const float *L = slut + g * W * CARD;
                float lb = 0.f;
#pragma unroll
                for (int s2 = 0; s2 < W; s2++) lb += L[s2 * CARD + byte_of(cl, s2)];
                if (lb <= qc[g].T) alive |= 1u << g;
            }
            if (leaf >= c1) alive = 0;
            if (restr && alive) {  // overflow rounds: the leaf must meet this slot's position range
                const uint32_t p0 = leaf * LEAF, p1 = min(p0 + LEAF, N);
#pragma unroll
                for (int g = 0; g < G; g++)
                    if (!(p0 < r1[g] && p1 > r0[g])) alive &= ~(1u << g);
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, alive != 0);
            if (bal) {
                uint32_t off = 0;
                if (lane == 0) off = atomicAdd(&wl_cnt, (uint32_t)__popc(bal));
                off = __shfl_sync(0xffffffffu, off, 0);
                if (alive) worklist[off + __popc(bal & lt)] = (leaf - c0) | (alive << 16);
            }
        }
        __syncthreads();
        // ---- phase B: the members of surviving leaves; two leaves' words in flight per warp
        const uint32_t nwl = wl_cnt;
        for (uint32_t e = warp * 2; e < nwl; e += 2 * NW) {
            uint32_t ent[2];
            uint4 wv[2][2];
#pragma unroll
            for (int k = 0; k < 2; k++) {
                ent[k] = e + k < nwl ? worklist[e + k] : 0;
                const uint32_t base = (c0 + (ent[k] & 0xFFFFu)) * LEAF;
#pragma unroll
                for (int u = 0; u < 2; u++) {
                    const uint32_t pos = base + u * 32 + lane;
                    wv[k][u] = (e + k < nwl && pos < N) ? ld_stream(sax + pos) : make_uint4(0, 0, 0, 0);
                }
            }
#pragma unroll
            for (int k = 0; k < 2; k++) {
                if (e + k >= nwl) break;
                const uint32_t am = ent[k] >> 16;
                const uint32_t base = (c0 + (ent[k] & 0xFFFFu)) * LEAF;
                loads++;
                if (lane < G && ((am >> lane) & 1u)) atomicAdd(&alive_cnt[lane], 1u);
#pragma unroll
                for (int g = 0; g < G; g++) {
                    if (!((am >> g) & 1u)) continue;
                    const QConst kq = qc[g];
                    const float *L = slut + g * W * CARD;
#pragma unroll
                    for (int u = 0; u < 2; u++) {
                        const uint32_t pos = base + u * 32 + lane;
                        const uint32_t v[4] = {wv[k][u].x, wv[k][u].y, wv[k][u].z, wv[k][u].w};
                        float lb = 0.f;
#pragma unroll
                        for (int s2 = 0; s2 < W; s2++) lb += L[s2 * CARD + byte_of(v, s2)];
                        bool keep = pos < N && lb <= kq.T && (pos < kq.ws || pos >= kq.we);
                        if (restr) keep = keep && pos >= r0[g] && pos < r1[g];
                        emit(keep, pos, g, qid[g], lane, lt, cbuf, cb_cnt, cand, cand_cnt, cap);
                    }
                }
            }
        }
        __syncthreads();
        if (t == 0) wl_cnt = 0;
        }
    }
    if (g0 != 0xffffffffu) flush();
    if (lane == 0 && loads) atomicAdd(leaf_loads, (unsigned long long)loads);
}

template <int G>
static void launch_leaf(const isax_index *ix, uint32_t nq, const uint32_t *qmap, const uint32_t *qrange, uint32_t lo,
                        uint32_t hi, float onepd, cudaStream_t s) {
    const size_t smem = (size_t)G * W * CARD * sizeof(float) + (size_t)G * CBUF * sizeof(uint32_t) + CHUNK * 4;
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
    const uint32_t nleaf = leaf_hi - leaf_lo;
    // chunk: as large as possible (fewer phase barriers) while leaving >= 8 tasks per SM for balance
    uint32_t chunk = CHUNK;
    while (chunk > 512 && (uint64_t)groups * ((nleaf + chunk - 1) / chunk) < 8ull * sms) chunk >>= 1;
    const uint64_t tasks = (uint64_t)groups * ((nleaf + chunk - 1) / chunk);
    const unsigned grid = (unsigned)std::max<uint64_t>(1, umin64(tasks, (uint64_t)sms));
    const QueryScratch &qs = ix->qs;
    cudaMemsetAsync(qs.task_ctr, 0, sizeof(uint32_t), s);
    leafscan_kernel<G><<<grid, LF_THREADS, smem, s>>>(
        reinterpret_cast<const uint4 *>(ix->sax), ix->lmeta, (uint32_t)ix->N, qs.lut, qs.qsax, qmap, qrange, nq,
        leaf_lo, leaf_hi, chunk, qs.bsf, qs.win, onepd, qs.cand, qs.cand_cnt, qs.cand_cap, qs.counters_leaf,
        qs.leaf_loads, qs.task_ctr);
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
