// isax_device.cuh: device helpers shared by the libisax kernels (iSAX symbol, key, compare).
#pragma once
#include "isax_internal.cuh"

namespace isax {

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// Number of beta_k <= m over the 255 breakpoints in `beta` (the tie goes up: S:90, R4).
__device__ __forceinline__ uint32_t sax_symbol(const double *beta, double m) {
    uint32_t c = 0;
#pragma unroll
    for (uint32_t step = 128; step >= 1; step >>= 1)
        if (beta[c + step - 1] <= m) c += step;
    return c;
}

// Plane-major bit interleave (R6): key bit (127 - 16p - s) = bit (7 - p) of symbol s.
// key.w holds planes 0,1 (most significant), key.x holds planes 6,7.
__device__ __forceinline__ uint4 isax_key(const uint32_t sym[W]) {
    uint32_t plane[8];
#pragma unroll
    for (int p = 0; p < 8; p++) {
        uint32_t v = 0;
#pragma unroll
        for (int s = 0; s < W; s++) v |= ((sym[s] >> (7 - p)) & 1u) << (15 - s);
        plane[p] = v;
    }
    return make_uint4((plane[6] << 16) | plane[7], (plane[4] << 16) | plane[5], (plane[2] << 16) | plane[3],
                      (plane[0] << 16) | plane[1]);
}

__device__ __forceinline__ uint4 word_key(uint4 wv) {
    uint32_t sym[W];
    const uint32_t v[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
    for (int s = 0; s < W; s++) sym[s] = (v[s >> 2] >> (8 * (s & 3))) & 0xFFu;
    return isax_key(sym);
}

__device__ __forceinline__ bool key_less(uint4 a, uint4 b) {
    if (a.w != b.w) return a.w < b.w;
    if (a.z != b.z) return a.z < b.z;
    if (a.y != b.y) return a.y < b.y;
    return a.x < b.x;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float bsf_d2(unsigned long long p) { return __uint_as_float((uint32_t)(p >> 32)); }

// append a near tie (R9) of query q; the count keeps growing past the capacity, so the host
// sees an overflow and sizes the query's next list from it (api.cu)
__device__ __forceinline__ void near_append(const NearList &nl, uint32_t q, uint32_t id, uint32_t pos, float d2) {
    const uint32_t k = atomicAdd(&nl.cnt[q], 1u);
    ISAX_BOUND(id != 0xffffffffu);
    if (k < nl.cap[q]) nl.base[nl.off[q] + k] = NearEntry{id, pos, d2, 0};
}

// y = fp32_rne(fl64((x - mu) / sd)), the stored value of R2/R3, without a full fp64 division per
// element. q = (x - mu) * rcp, with rcp = fl64(1/sd), is within 2.5 fp64 ulps of the correctly
// rounded quotient Q. Rounding to fp32 drops the low 29 bits of the fp64 significand, and it can
// only change between q - 8 ulp and q + 8 ulp (>= 4 ulps even across a binade) when those bits lie
// within 8 of the halfway point 2^28. Outside that window, and with q a normal fp32 magnitude,
// fp32(q) is what Q rounds to too (Q lies between q - 8 ulp and q + 8 ulp, and rounding is
// monotone). Otherwise, about once in 1e7 elements, and for q = 0, the true division decides.
// The result equals the definition bit for bit.
__device__ __forceinline__ float znorm_value(float x, double mu, double sd, double rcp) {
    const double t = __dsub_rn((double)x, mu);
    const double q = __dmul_rn(t, rcp);
    const unsigned long long b = (unsigned long long)__double_as_longlong(q);
    const uint32_t ex = (uint32_t)(b >> 52) & 0x7FFu;          // biased exponent
    const uint32_t low = (uint32_t)b & ((1u << 29) - 1u);     // the bits fp32 rounding drops
    if (ex >= 898u && ex <= 1149u && low - ((1u << 28) - 8u) > 16u) return __double2float_rn(q);
    return __double2float_rn(__ddiv_rn(t, sd));
}

// exclusive prefix of the list lengths over q < Q into pre[0..Q], by the whole CTA. A list that
// overflowed (cand_cnt > cap) counts as empty: it holds an arbitrary subset of its query's
// candidates, and the query rescans the smallest bounds in its next round anyway (R10), so
// refining it now would be wasted reads.
template <int NT>
__device__ __forceinline__ void cand_prefix(const uint32_t *__restrict__ cand_cnt, uint32_t Q, uint32_t cap,
                                            uint32_t *pre) {
    __shared__ uint32_t wsum[NT / 32];
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    uint32_t carry = 0;
    for (uint32_t b = 0; b < Q; b += NT) {
        const uint32_t q = b + t;
        const uint32_t v = q < Q && cand_cnt[q] <= cap ? cand_cnt[q] : 0;
        uint32_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (uint32_t)o) inc += u;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        uint32_t wpre = 0, tot = 0;
        for (uint32_t w = 0; w < NT / 32; w++) {
            if (w < warp) wpre += wsum[w];
            tot += wsum[w];
        }
        if (q < Q) pre[q] = carry + wpre + inc - v;
        carry += tot;
        __syncthreads();
    }
    if (t == 0) pre[Q] = carry;
    __syncthreads();
}

}  // namespace isax
