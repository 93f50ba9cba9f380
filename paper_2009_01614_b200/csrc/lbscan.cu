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

void launch_lbscan(const isax_index *ix, uint32_t nq, const uint32_t *qmap, const uint32_t *qrange, uint32_t lo,
                   uint32_t hi, float delta, cudaStream_t s) {
    if (!nq || hi <= lo) return;
    const float onepd = 1.0f + delta;
    if (nq >= 4) launch_g<4>(ix, nq, qmap, qrange, lo, hi, onepd, s);
    else if (nq == 3) launch_g<3>(ix, nq, qmap, qrange, lo, hi, onepd, s);
    else if (nq == 2) launch_g<2>(ix, nq, qmap, qrange, lo, hi, onepd, s);
    else launch_g<1>(ix, nq, qmap, qrange, lo, hi, onepd, s);
}

}  // namespace isax
