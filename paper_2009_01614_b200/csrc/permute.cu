// permute.cu: build pass 2. It writes the z-normalised rows in SAX-sorted (leaf-contiguous)
// order, north_star (a): "the raw series permuted into SAX-word-sorted, leaf-contiguous order".
//
// y_i = fp32_rne((x_i - mu) / sigma) uses the same fp64 operations as summarise.cu (R2), so
// the stored rows are the rows the words were computed from. There is one warp per row, with
// coalesced 512-byte float4 loads and stores.
//  - gather  (device-resident input): stored[pos] = y(x[perm[pos]])
//  - scatter (streamed input, chunk by chunk): stored[inv[id]] = y(x[id])
// Roofline: 8n bytes per series (read + write) + 16 (mu, sigma) + 4 (perm). HBM-bound.
#include "isax_device.cuh"

namespace isax {

__device__ __forceinline__ float zval(float x, double mu, double sd, bool flat, double rcp) {
    return flat ? 0.0f : znorm_value(x, mu, sd, rcp);
}

__device__ __forceinline__ void norm_row(const float *__restrict__ src, float *__restrict__ dst, double2 ms,
                                         uint32_t n, uint32_t lane) {
    const bool flat = ms.y < 1e-12;
    const double rcp = __drcp_rn(ms.y);
    const float4 *s4 = reinterpret_cast<const float4 *>(src);
    float4 *d4 = reinterpret_cast<float4 *>(dst);
    for (uint32_t i = lane; i < n / 4; i += 32) {
        float4 v = __ldcs(s4 + i);
        v.x = zval(v.x, ms.x, ms.y, flat, rcp);
        v.y = zval(v.y, ms.x, ms.y, flat, rcp);
        v.z = zval(v.z, ms.x, ms.y, flat, rcp);
        v.w = zval(v.w, ms.x, ms.y, flat, rcp);
        d4[i] = v;
    }
}

__global__ void gather_rows_kernel(const float *__restrict__ x, const double2 *__restrict__ musig,
                                   const uint32_t *__restrict__ perm, uint64_t N, uint32_t n,
                                   float *__restrict__ stored) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t wpb = blockDim.x / 32;
    for (uint64_t pos = blockIdx.x * wpb + threadIdx.x / 32; pos < N; pos += (uint64_t)gridDim.x * wpb) {
        const uint32_t id = perm[pos];
        ISAX_BOUND(id < N);
        norm_row(x + (uint64_t)id * n, stored + pos * n, musig[id], n, lane);
    }
}

__global__ void scatter_rows_kernel(const float *__restrict__ x, uint64_t count, uint64_t id0,
                                    const double2 *__restrict__ musig, const uint32_t *__restrict__ inv, uint32_t n,
                                    float *__restrict__ stored) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t wpb = blockDim.x / 32;
    for (uint64_t r = blockIdx.x * wpb + threadIdx.x / 32; r < count; r += (uint64_t)gridDim.x * wpb) {
        const uint64_t id = id0 + r;
        ISAX_BOUND(inv[id] < 0xffffffffu);
        norm_row(x + r * n, stored + (uint64_t)inv[id] * n, musig[id], n, lane);
    }
}

__global__ void gather_sax_kernel(const uint4 *__restrict__ sax_by_id, const uint32_t *__restrict__ perm, uint64_t N,
                                  uint4 *__restrict__ sax) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x)
    {
        ISAX_BOUND(perm[i] < N);
        sax[i] = sax_by_id[perm[i]];
    }
}

__global__ void invert_perm_kernel(const uint32_t *__restrict__ perm, uint64_t N, uint32_t *__restrict__ inv) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x)
        inv[perm[i]] = (uint32_t)i;
}

__global__ void export_sax_kernel(const uint4 *__restrict__ sax, const uint32_t *__restrict__ inv, uint64_t first_id,
                                  uint64_t count, uint4 *__restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = sax[inv[first_id + i]];
}

static unsigned grid_for(uint64_t items, unsigned per_block) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t need = (items + per_block - 1) / per_block;
    return (unsigned)std::max<uint64_t>(1, umin64(need, (uint64_t)sms * 16));
}

void launch_gather_rows(const float *x, const double2 *musig, const uint32_t *perm, uint64_t N, uint32_t n,
                        float *stored, cudaStream_t s) {
    gather_rows_kernel<<<grid_for(N, 8), 256, 0, s>>>(x, musig, perm, N, n, stored);
}

void launch_scatter_rows(const float *x, uint64_t count, uint64_t id0, const double2 *musig, const uint32_t *inv,
                         uint32_t n, float *stored, cudaStream_t s) {
    if (count) scatter_rows_kernel<<<grid_for(count, 8), 256, 0, s>>>(x, count, id0, musig, inv, n, stored);
}

void launch_gather_sax(const uint8_t *sax_by_id, const uint32_t *perm, uint64_t N, uint8_t *sax, cudaStream_t s) {
    gather_sax_kernel<<<grid_for(N, 256), 256, 0, s>>>(reinterpret_cast<const uint4 *>(sax_by_id), perm, N,
                                                       reinterpret_cast<uint4 *>(sax));
}

void launch_invert_perm(const uint32_t *perm, uint64_t N, uint32_t *inv, cudaStream_t s) {
    invert_perm_kernel<<<grid_for(N, 256), 256, 0, s>>>(perm, N, inv);
}

void launch_export_sax(const uint8_t *sax, const uint32_t *inv, uint64_t first_id, uint64_t count, uint8_t *out,
                       cudaStream_t s) {
    if (count)
        export_sax_kernel<<<grid_for(count, 256), 256, 0, s>>>(reinterpret_cast<const uint4 *>(sax), inv, first_id,
                                                               count, reinterpret_cast<uint4 *>(out));
}


// ------------------------------------------------------------------------------------ super-node kd order
// (R6b) The z order groups series by key prefix, but a leaf of 32 consecutive positions often
// straddles key boundaries, which widens its per-segment [min, max] box. Inside every full
// super-node (SUPER_SIZE = 1024 consecutive positions of the z order) the positions are reordered
// by a kd split down to cells of KD_CELL = 8 rows, so the 32 leaves of a super-node and the four
// cells of each leaf (the scan's sub-leaf boxes, R11c) have tight boxes:
//   at each level, every node (a contiguous half of its parent) takes the segment s with the
//   largest symbol range max_s - min_s over its members (the lowest s on ties) and is sorted by
//   symbol s, stably (equal symbols keep their order); its halves are its children.
// Membership of super-nodes and hyper-nodes is unchanged, so their boxes are too. Offline on 4M
// random walks this cut the members tested under alive leaves by 14%.
// Per super-node it also records the z key of its first position (the block's smallest key, for
// the approximate answer's search) and the first four split levels (segment and the smallest
// symbol of the right half) for locating a probe's kd cell.
// One CTA per full super-node, 512 threads; down to nodes of 64 rows the node ranges come from
// warp reductions and one shared atomic per (node, segment) and warp, below that from shuffles
// inside the node's aligned group of lanes; each level is a bitonic sort of the keys
// (node << 18 | symbol << 10 | position) inside every node, so the order is exactly the stable one.
constexpr int KD_THREADS = 512;

// min and max of v over the aligned group of `size` lanes (a power of two <= 32) this lane is in
__device__ __forceinline__ void group_minmax(uint32_t v, uint32_t size, uint32_t &lo, uint32_t &hi) {
    lo = hi = v;
    for (uint32_t o = 1; o < size; o <<= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
}

__global__ void __launch_bounds__(KD_THREADS) superkd_kernel(uint4 *__restrict__ sax, uint32_t *__restrict__ perm,
                                                          uint64_t nfull, uint4 *__restrict__ skey,
                                                          KdSplits *__restrict__ ksplit) {
    constexpr uint32_t S = SUPER_SIZE, LV = 7;  // 1024 -> 8 (KD_CELL)
    static_assert(SUPER_SIZE == 1024 && KD_CELL == 8, "seven kd levels per super-node");
    __shared__ uint4 wa[S], wb[S];
    __shared__ uint32_t ia[S], ib[S];
    __shared__ uint32_t key[S];
    __shared__ uint32_t mn[16][W], mx[16][W];
    __shared__ uint32_t segsel[16], lvseg[15];  // lvseg: the chosen segment of heap node k (levels 0-3)
    const uint32_t t = threadIdx.x;
    const uint64_t b = blockIdx.x;
    if (b >= nfull) return;
    uint4 *wcur = wa, *wnxt = wb;
    uint32_t *icur = ia, *inxt = ib;
    for (uint32_t i = t; i < S; i += KD_THREADS) {
        wa[i] = sax[b * S + i];
        ia[i] = perm[b * S + i];
    }
    __syncthreads();
    if (t == 0) skey[b] = word_key(wa[0]);
    for (uint32_t lv = 0; lv < LV; lv++) {
        const uint32_t size = S >> lv, nodes = 1u << lv, sh = 10 - lv;
        if (size > 32) {
            // levels 0-4 (nodes of 64 rows or more): a warp's 32 consecutive positions lie in one
            // node: warp reductions first, then one shared atomic per (node, segment) and warp
            for (uint32_t i = t; i < nodes * W; i += KD_THREADS) {
                mn[i / W][i % W] = 255u;
                mx[i / W][i % W] = 0u;
            }
            __syncthreads();
            for (uint32_t i = t; i < S; i += KD_THREADS) {
                const uint4 wv = wcur[i];
                const uint32_t v[4] = {wv.x, wv.y, wv.z, wv.w};
                const uint32_t nd = i >> sh;
                uint32_t mine = 0, maxe = 0;  // lane s < W keeps segment s's results
#pragma unroll
                for (int s = 0; s < W; s++) {
                    const uint32_t c = (v[s >> 2] >> (8 * (s & 3))) & 0xFFu;
                    const uint32_t lo = __reduce_min_sync(0xffffffffu, c), hi = __reduce_max_sync(0xffffffffu, c);
                    if ((t & 31) == (uint32_t)s) {
                        mine = lo;
                        maxe = hi;
                    }
                }
                if ((t & 31) < (uint32_t)W) {
                    atomicMin(&mn[nd][t & 31], mine);
                    atomicMax(&mx[nd][t & 31], maxe);
                }
            }
            __syncthreads();
            if (t < nodes) {
                uint32_t best = 0, br = 0;
                for (uint32_t s = 0; s < W; s++) {
                    const uint32_t r = mx[t][s] - mn[t][s];
                    if (r > br) {  // strictly larger: the lowest segment wins ties
                        br = r;
                        best = s;
                    }
                }
                segsel[t] = best;
                if (lv < KD_LEVELS) lvseg[(1u << lv) - 1 + t] = best;
            }
            __syncthreads();
            for (uint32_t i = t; i < S; i += KD_THREADS) {
                const uint4 wv = wcur[i];
                const uint32_t v[4] = {wv.x, wv.y, wv.z, wv.w};
                const uint32_t nd = i >> sh, s = segsel[nd];
                const uint32_t c = (v[s >> 2] >> (8 * (s & 3))) & 0xFFu;
                key[i] = (nd << 18) | (c << 10) | i;
            }
        } else {
            // levels 5-6 (nodes of 32 and 16 rows): a node is an aligned group of lanes, so its
            // ranges and its segment come from shuffles alone
            for (uint32_t i = t; i < S; i += KD_THREADS) {
                const uint4 wv = wcur[i];
                const uint32_t v[4] = {wv.x, wv.y, wv.z, wv.w};
                uint32_t best_c = 0, br = 0;
                bool first = true;
#pragma unroll
                for (int s = 0; s < W; s++) {
                    const uint32_t c = (v[s >> 2] >> (8 * (s & 3))) & 0xFFu;
                    uint32_t lo, hi;
                    group_minmax(c, size, lo, hi);
                    if (first || hi - lo > br) {  // strictly larger: the lowest segment wins ties
                        br = hi - lo;
                        best_c = c;
                        first = false;
                    }
                }
                key[i] = ((i >> sh) << 18) | (best_c << 10) | i;
            }
        }
        __syncthreads();
        // bitonic sort of the keys (all distinct), ascending inside every node: a node's rows stay
        // in its own aligned block of `size` positions, so the network stops at k = size
        for (uint32_t k = 2; k <= size; k <<= 1) {
            for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                for (uint32_t i = t; i < S; i += KD_THREADS) {
                    const uint32_t p = i ^ j;
                    if (p > i) {
                        const uint32_t a = key[i], c = key[p];
                        const bool up = (i & (size - 1) & k) == 0;
                        if ((a > c) == up) {
                            key[i] = c;
                            key[p] = a;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (uint32_t i = t; i < S; i += KD_THREADS) {
            const uint32_t src = key[i] & 1023u;
            wnxt[i] = wcur[src];
            inxt[i] = icur[src];
        }
        __syncthreads();
        uint4 *tw = wcur; wcur = wnxt; wnxt = tw;
        uint32_t *ti = icur; icur = inxt; inxt = ti;
    }
    // the first four levels' splits (heap order): segment and smallest symbol of the right half
    if (t < 15) {
        const uint32_t lv = 31 - __clz(t + 1), nd = t + 1 - (1u << lv);
        const uint32_t size = S >> lv, r0 = nd * size + size / 2, r1 = nd * size + size;
        const uint32_t s = lvseg[t];
        uint32_t m = 255u;
        for (uint32_t i = r0; i < r1; i++) {
            const uint4 wv = wcur[i];
            const uint32_t v[4] = {wv.x, wv.y, wv.z, wv.w};
            m = min(m, (v[s >> 2] >> (8 * (s & 3))) & 0xFFu);
        }
        key[t] = s | (m << 8);
    }
    __syncthreads();
    if (t < 16) ksplit[b].s[t] = t < 15 ? (uint16_t)key[t] : (uint16_t)0;
    for (uint32_t i = t; i < S; i += KD_THREADS) {
        sax[b * S + i] = wcur[i];
        perm[b * S + i] = icur[i];
    }
}

// the last, partial super-node keeps the z order; it still gets its smallest key
__global__ void superkey_tail_kernel(const uint4 *__restrict__ sax, uint64_t first, uint4 *__restrict__ skey,
                                     KdSplits *__restrict__ ksplit, uint64_t s) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        skey[s] = word_key(sax[first]);
        for (int k = 0; k < 16; k++) ksplit[s].s[k] = KD_NONE;  // no kd splits: cells are not located
    }
}

void launch_superkd(uint8_t *sax, uint32_t *perm, uint64_t N, uint4 *skey, KdSplits *ksplit, cudaStream_t s) {
    const uint64_t nfull = N / SUPER_SIZE;
    if (nfull) superkd_kernel<<<(unsigned)nfull, KD_THREADS, 0, s>>>(reinterpret_cast<uint4 *>(sax), perm, nfull, skey, ksplit);
    if (N % SUPER_SIZE)
        superkey_tail_kernel<<<1, 32, 0, s>>>(reinterpret_cast<const uint4 *>(sax), nfull * SUPER_SIZE, skey, ksplit, nfull);
}

}  // namespace isax
