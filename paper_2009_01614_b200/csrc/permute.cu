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
        norm_row(x + r * n, stored + (uint64_t)inv[id] * n, musig[id], n, lane);
    }
}

__global__ void gather_sax_kernel(const uint4 *__restrict__ sax_by_id, const uint32_t *__restrict__ perm, uint64_t N,
                                  uint4 *__restrict__ sax) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x)
        sax[i] = sax_by_id[perm[i]];
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

}  // namespace isax
