// sort.cu: stable LSD radix sort of (128-bit key, u32 id) pairs. It gives the canonical
// SAX-sorted order (R6).
//
// It replaces the paper's RecBuf / iSAX-buffer insertion keyed by the w first bits
// and the per-subtree construction. The top 16 key bits
// are exactly that root-subtree key, and the sort orders the rest of each subtree by its
// plane-interleaved word, so every node of a round-robin-split tree is a contiguous range.
//
// It makes 16 passes of 8-bit digits from least significant. Each pass is histogram ->
// exclusive scan (digit-major) -> stable scatter. The input ids are iota, and every pass is
// stable, so equal keys keep ascending id order: the order is ascending (key, id), with no
// tie-break work.
// Stability inside a block: items are taken in rounds of 256 (thread order). Ranks inside a
// warp come from __match_any_sync, and warp offsets from a per-digit prefix over warps.
#include "isax_device.cuh"

namespace isax {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;

__device__ __forceinline__ uint32_t digit_of(const uint4 &k, int pass) {
    const uint32_t w = pass < 4 ? k.x : pass < 8 ? k.y : pass < 12 ? k.z : k.w;
    return (w >> ((pass & 3) * 8)) & 0xFFu;
}

__global__ void __launch_bounds__(RS_THREADS) rs_hist(const uint4 *__restrict__ keys, uint64_t N,
                                                      uint64_t per_block, int pass, uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t b0 = (uint64_t)blockIdx.x * per_block;
    const uint64_t b1 = umin64(N, b0 + per_block);
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t base = b0; base < b1; base += RS_THREADS) {
        const uint64_t i = base + threadIdx.x;
        const bool valid = i < b1;
        const uint32_t d = valid ? digit_of(keys[i], pass) : 256u + lane;
        const uint32_t m = __match_any_sync(0xffffffffu, d);
        if (valid && lane == (uint32_t)(__ffs(m) - 1)) atomicAdd(&h[d], (uint32_t)__popc(m));
    }
    __syncthreads();
    hist[(uint64_t)threadIdx.x * gridDim.x + blockIdx.x] = h[threadIdx.x];
}

// Per-digit exclusive scan over the blocks: CTA d scans hist[d][0..nb) in place and writes the
// digit total. The scatter adds the exclusive prefix of the totals (its own 256-entry scan).
constexpr int SC_THREADS = 1024;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t *tot) {
    __shared__ uint32_t ws[32];
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (uint32_t)o) inc += u;
    }
    if (lane == 31) ws[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t nw = blockDim.x / 32;
        uint32_t x = lane < nw ? ws[lane] : 0, xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= (uint32_t)o) xi += u;
        }
        if (lane < nw) ws[lane] = xi - x;
        if (lane == nw - 1 && tot) *tot = xi;
    }
    __syncthreads();
    const uint32_t r = ws[warp] + inc - v;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(SC_THREADS) rs_scan_digits(uint32_t *__restrict__ hist, uint32_t nb,
                                                             uint32_t *__restrict__ dtotal) {
    __shared__ uint32_t total;
    const uint32_t d = blockIdx.x;
    uint32_t *h = hist + (uint64_t)d * nb;
    const uint32_t per = (nb + SC_THREADS - 1) / SC_THREADS;
    const uint32_t s0 = threadIdx.x * per, s1 = min(nb, s0 + per);
    uint32_t sum = 0;
    for (uint32_t i = s0; i < s1; i++) sum += h[i];
    uint32_t run = block_exclusive_scan(sum, &total);
    for (uint32_t i = s0; i < s1; i++) {
        const uint32_t v = h[i];
        h[i] = run;
        run += v;
    }
    __syncthreads();
    if (threadIdx.x == 0) dtotal[d] = total;
}

__global__ void __launch_bounds__(RS_THREADS) rs_scatter(const uint4 *__restrict__ kin, const uint32_t *__restrict__ vin,
                                                         uint4 *__restrict__ kout, uint32_t *__restrict__ vout,
                                                         uint64_t N, uint64_t per_block, int pass,
                                                         const uint32_t *__restrict__ offs,
                                                         const uint32_t *__restrict__ dtotal) {
    __shared__ uint32_t base[256];
    __shared__ uint32_t wcnt[RS_WARPS][256];
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t doff = block_exclusive_scan(dtotal[t], nullptr);  // start of digit t's output
    base[t] = doff + offs[(uint64_t)t * gridDim.x + blockIdx.x];
#pragma unroll
    for (int w = 0; w < RS_WARPS; w++) wcnt[w][t] = 0;
    __syncthreads();
    const uint64_t b0 = (uint64_t)blockIdx.x * per_block;
    const uint64_t b1 = umin64(N, b0 + per_block);
    const uint32_t lt = (1u << lane) - 1u;
    for (uint64_t r = b0; r < b1; r += RS_THREADS) {
        const uint64_t i = r + t;
        const bool valid = i < b1;
        uint4 k = make_uint4(0, 0, 0, 0);
        uint32_t v = 0;
        if (valid) {
            k = kin[i];
            v = vin[i];
        }
        const uint32_t d = valid ? digit_of(k, pass) : 256u + lane;
        const uint32_t m = __match_any_sync(0xffffffffu, d);
        const uint32_t rank = __popc(m & lt);
        if (valid && rank == 0) wcnt[warp][d] = __popc(m);
        __syncthreads();
        {  // thread t owns digit t: running offsets over warps, in warp order
            uint32_t run = base[t];
#pragma unroll
            for (int w = 0; w < RS_WARPS; w++) {
                const uint32_t c = wcnt[w][t];
                wcnt[w][t] = run;
                run += c;
            }
            base[t] = run;
        }
        __syncthreads();
        if (valid) {
            const uint32_t dst = wcnt[warp][d] + rank;
            ISAX_BOUND(dst < N);
            kout[dst] = k;
            vout[dst] = v;
        }
        __syncthreads();
#pragma unroll
        for (int w = 0; w < RS_WARPS; w++) wcnt[w][t] = 0;
        __syncthreads();
    }
}

__global__ void iota_kernel(uint32_t *ids, uint64_t N) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x)
        ids[i] = (uint32_t)i;
}

int radix_sort_keys(uint4 *keys, uint32_t *ids, uint64_t N, uint32_t *perm_out, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    iota_kernel<<<sms * 8, 256, 0, s>>>(ids, N);
    const uint64_t nb = std::max<uint64_t>(1, umin64((N + RS_THREADS - 1) / RS_THREADS, (uint64_t)sms * 8));
    const uint64_t per_block = (N + nb - 1) / nb;
    uint4 *k2 = nullptr;
    uint32_t *hist = nullptr;
    ISAX_CUDA(cudaMalloc(&k2, N * sizeof(uint4)));
    cudaError_t e = cudaMalloc(&hist, (nb * 256 + 256) * sizeof(uint32_t));
    if (e != cudaSuccess) {
        cudaFree(k2);
        return cuda_error(e, "cudaMalloc(sort hist)");
    }
    uint4 *ka = keys, *kb = k2;
    uint32_t *va = ids, *vb = perm_out;
    for (int pass = 0; pass < 16; pass++) {
        rs_hist<<<(unsigned)nb, RS_THREADS, 0, s>>>(ka, N, per_block, pass, hist);
        rs_scan_digits<<<256, SC_THREADS, 0, s>>>(hist, (uint32_t)nb, hist + nb * 256);
        rs_scatter<<<(unsigned)nb, RS_THREADS, 0, s>>>(ka, va, kb, vb, N, per_block, pass, hist, hist + nb * 256);
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    // 16 passes (even): the result is back in (keys, ids). Copy ids into perm_out.
    cudaMemcpyAsync(perm_out, va, N * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
    e = cudaStreamSynchronize(s);
    cudaFree(k2);
    cudaFree(hist);
    if (e != cudaSuccess) return cuda_error(e, "radix sort");
    return ISAX_OK;
}

}  // namespace isax
