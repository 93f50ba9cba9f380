// summarise.cu: build pass 1, z-norm -> PAA -> SAX -> 128-bit key, one series per thread.
//
// Method: P:168 (PAA, iSAX symbols); P:213-222 / P:293-296 (bulk summarisation by the index
// workers); P:216-217 (root subtree = the first bit of each segment). Readings R2-R4 and R6
// (DESIGN.md).
//
// Precision (R3): mu, sigma and each PAA mean are fp64 sums taken strictly left to right over
// the points of one series, with no FMA contraction (explicit __d*_rn intrinsics). That is the
// plain definition, so the words match the oracle bit for bit, independent of launch shape.
// The order of a sum is per series, so each thread owns one series, and a warp stages its 32
// rows in shared memory with coalesced 512-byte loads. The stride is padded to n+1 words, so
// the per-thread sequential reads are bank-conflict free (bank = (lane + i) mod 32).
//
// Roofline: 4n bytes read + 16 (word) + 16 (key) + 16 (mu, sigma) bytes written per series;
// ~4n fp64 ops. HBM-bound at n=256 if fp64 latency chains are hidden by enough warps (6 per SM).
#include "isax_device.cuh"

namespace isax {

#include "breakpoints.inc"

__constant__ double c_beta[ISAX_NBETA] = ISAX_BETA_INIT;

// NT = n when the kernel is specialised for it (index math by a constant), 0 = generic n.
template <uint32_t NT>
__global__ void __launch_bounds__(32) summarise_kernel(const float *__restrict__ x, uint64_t count, uint32_t n_rt,
                                                         uint64_t id0, uint8_t *__restrict__ sax_by_id,
                                                         uint4 *__restrict__ key, double2 *__restrict__ musig,
                                                         uint32_t *__restrict__ bad) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *beta = reinterpret_cast<double *>(smem_raw);
    double2 *ms = reinterpret_cast<double2 *>(smem_raw + ISAX_NBETA * sizeof(double) + 8);  // [32] (mu, sigma)
    float *rows = reinterpret_cast<float *>(ms + 32);
    const uint32_t n = NT ? NT : n_rt;
    const uint32_t lane = threadIdx.x;
    const uint32_t stride = n + 1;  // bank = (lane + i) mod 32 for the per-thread sequential reads
    for (uint32_t k = lane; k < ISAX_NBETA; k += 32) beta[k] = c_beta[k];
    const uint32_t seg = n / W;
    const uint32_t per_row = n / 4;
    const uint64_t ngroups = (count + 31) / 32;
    for (uint64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const uint64_t r0 = g * 32;
        const uint32_t nrows = (uint32_t)umin64(32, count - r0);
        __syncwarp();
        // stage the 32 rows (contiguous in memory): lane l moves float4 e = l, l+32, ... of the
        // tile, 16 loads in flight per lane before the shared stores (each warp instruction reads
        // 512 contiguous bytes)
        {
            const uint32_t total = nrows * per_row;
            const float4 *src = reinterpret_cast<const float4 *>(x + r0 * n);
            constexpr uint32_t B = 16;
            for (uint32_t e0 = 0; e0 < total; e0 += 32 * B) {
                float4 v[B];
#pragma unroll
                for (uint32_t k = 0; k < B; k++) {
                    const uint32_t e = e0 + k * 32 + lane;
                    if (e < total) v[k] = __ldcs(src + e);
                }
#pragma unroll
                for (uint32_t k = 0; k < B; k++) {
                    const uint32_t e = e0 + k * 32 + lane;
                    if (e < total) {
                        float *d = rows + (e / per_row) * stride + 4 * (e % per_row);
                        d[0] = v[k].x; d[1] = v[k].y; d[2] = v[k].z; d[3] = v[k].w;
                    }
                }
            }
        }
        __syncwarp();
        bool finite = true;
        if (lane < nrows) {
            const float *row = rows + lane * stride;
            // C1: mu and sigma, left to right (R2, R3). These two chains are the only sequential
            // parts; the loops are unrolled so the shared loads run ahead of the add chain.
            double s = 0.0;
#pragma unroll 16
            for (uint32_t i = 0; i < n; i++) {
                const float v = row[i];
                finite &= isfinite(v);
                s = __dadd_rn(s, (double)v);
            }
            const double mu = __ddiv_rn(s, (double)n);
            double s2 = 0.0;
#pragma unroll 16
            for (uint32_t i = 0; i < n; i++) {
                const double t = __dsub_rn((double)row[i], mu);
                s2 = __dadd_rn(s2, __dmul_rn(t, t));
            }
            ms[lane] = make_double2(mu, __dsqrt_rn(__ddiv_rn(s2, (double)n)));
        }
        __syncwarp();
        // y = fp32((x - mu) / sigma) for the whole tile, warp-cooperatively: the divisions are
        // independent, so all 32 lanes stream them with full ILP; y overwrites x in place
        double rcp = 0.0;
        if (lane < nrows) rcp = __drcp_rn(ms[lane].y);
        for (uint32_t r = 0; r < nrows; r++) {
            const double2 m = ms[r];
            const double rr = __shfl_sync(0xffffffffu, rcp, r);
            float *p = rows + r * stride;
#pragma unroll 4
            for (uint32_t c = lane; c < n; c += 32)
                p[c] = m.y < 1e-12 ? 0.0f : znorm_value(p[c], m.x, m.y, rr);
        }
        __syncwarp();
        if (lane < nrows) {
            const float *row = rows + lane * stride;
            // C2: the 16 segment sums, left to right within each segment, interleaved across segments
            double acc[W];
#pragma unroll
            for (int sg = 0; sg < W; sg++) acc[sg] = 0.0;
            for (uint32_t j = 0; j < seg; j++) {
#pragma unroll
                for (int sg = 0; sg < W; sg++) acc[sg] = __dadd_rn(acc[sg], (double)row[sg * seg + j]);
            }
            // C4: symbols, 16 independent binary searches
            uint32_t sym[W];
#pragma unroll
            for (int sg = 0; sg < W; sg++) sym[sg] = sax_symbol(beta, __ddiv_rn(acc[sg], (double)seg));
            const uint64_t id = id0 + r0 + lane;
            uint4 wv;
            wv.x = sym[0] | (sym[1] << 8) | (sym[2] << 16) | (sym[3] << 24);
            wv.y = sym[4] | (sym[5] << 8) | (sym[6] << 16) | (sym[7] << 24);
            wv.z = sym[8] | (sym[9] << 8) | (sym[10] << 16) | (sym[11] << 24);
            wv.w = sym[12] | (sym[13] << 8) | (sym[14] << 16) | (sym[15] << 24);
            reinterpret_cast<uint4 *>(sax_by_id)[id] = wv;
            key[id] = isax_key(sym);
            musig[id] = ms[lane];
            if (!finite) atomicOr(bad, 1u);
        }
    }
}

// Half-row staging for n = 128 and 256: the warp stages its 32 rows half a row at a time (16.5 KB
// instead of 33 KB of shared memory), so twice as many warps fit on an SM and twice as many
// sequential fp64 chains are in flight. Each pass (mean, variance, then y and the segment sums)
// restages both halves; the second and third reads of a half come from L2. The fp64 operations
// and their order per series are those of summarise_kernel (R3): identical words.
template <uint32_t NT>
__global__ void __launch_bounds__(32) summarise_half_kernel(const float *__restrict__ x, uint64_t count, uint64_t id0,
                                                            uint8_t *__restrict__ sax_by_id, uint4 *__restrict__ key,
                                                            double2 *__restrict__ musig, uint32_t *__restrict__ bad) {
    constexpr uint32_t n = NT, P = NT / 2, seg = NT / W, SPP = W / 2;  // columns and segments per half
    constexpr uint32_t stride = P + 1;                                  // bank = (lane + i) mod 32
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *beta = reinterpret_cast<double *>(smem_raw);
    double2 *ms = reinterpret_cast<double2 *>(smem_raw + ISAX_NBETA * sizeof(double) + 8);
    float *rows = reinterpret_cast<float *>(ms + 32);
    const uint32_t lane = threadIdx.x;
    for (uint32_t k = lane; k < ISAX_NBETA; k += 32) beta[k] = c_beta[k];
    const uint64_t ngroups = (count + 31) / 32;
    for (uint64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const uint64_t r0 = g * 32;
        const uint32_t nrows = (uint32_t)umin64(32, count - r0);
        // half h of the 32 rows into shared memory (each row's half is P contiguous floats)
        auto stage = [&](uint32_t h) {
            __syncwarp();
            constexpr uint32_t per = P / 4;
            const uint32_t total = nrows * per;
            constexpr uint32_t B = 8;
            for (uint32_t e0 = 0; e0 < total; e0 += 32 * B) {
                float4 v[B];
#pragma unroll
                for (uint32_t k = 0; k < B; k++) {
                    const uint32_t e = e0 + k * 32 + lane;
                    if (e < total) v[k] = __ldg(reinterpret_cast<const float4 *>(x + (r0 + e / per) * n + h * P) + e % per);
                }
#pragma unroll
                for (uint32_t k = 0; k < B; k++) {
                    const uint32_t e = e0 + k * 32 + lane;
                    if (e < total) {
                        float *d = rows + (e / per) * stride + 4 * (e % per);
                        d[0] = v[k].x; d[1] = v[k].y; d[2] = v[k].z; d[3] = v[k].w;
                    }
                }
            }
            __syncwarp();
        };
        const float *row = rows + lane * stride;
        bool finite = true;
        double s = 0.0;  // C1, left to right over both halves (R2, R3)
#pragma unroll
        for (uint32_t h = 0; h < 2; h++) {
            stage(h);
            if (lane < nrows) {
#pragma unroll 16
                for (uint32_t i = 0; i < P; i++) {
                    const float v = row[i];
                    finite &= isfinite(v);
                    s = __dadd_rn(s, (double)v);
                }
            }
        }
        const double mu = __ddiv_rn(s, (double)n);
        double s2 = 0.0;
#pragma unroll
        for (uint32_t h = 0; h < 2; h++) {
            stage(h);
            if (lane < nrows) {
#pragma unroll 16
                for (uint32_t i = 0; i < P; i++) {
                    const double t = __dsub_rn((double)row[i], mu);
                    s2 = __dadd_rn(s2, __dmul_rn(t, t));
                }
            }
        }
        if (lane < nrows) ms[lane] = make_double2(mu, __dsqrt_rn(__ddiv_rn(s2, (double)n)));
        double rcp = 0.0;
        __syncwarp();
        if (lane < nrows) rcp = __drcp_rn(ms[lane].y);
        double acc[W];
#pragma unroll
        for (int sg = 0; sg < W; sg++) acc[sg] = 0.0;
#pragma unroll
        for (uint32_t h = 0; h < 2; h++) {
            stage(h);
            // y = fp32((x - mu) / sigma) for the half tile, warp-cooperatively, in place
            for (uint32_t r = 0; r < nrows; r++) {
                const double2 m = ms[r];
                const double rr = __shfl_sync(0xffffffffu, rcp, r);
                float *pr = rows + r * stride;
#pragma unroll 4
                for (uint32_t c = lane; c < P; c += 32) pr[c] = m.y < 1e-12 ? 0.0f : znorm_value(pr[c], m.x, m.y, rr);
            }
            __syncwarp();
            if (lane < nrows) {  // C2: this half's segments, left to right within each
                for (uint32_t j = 0; j < seg; j++) {
#pragma unroll
                    for (uint32_t sg = 0; sg < SPP; sg++)
                        acc[h * SPP + sg] = __dadd_rn(acc[h * SPP + sg], (double)row[sg * seg + j]);
                }
            }
        }
        if (lane < nrows) {
            uint32_t sym[W];
#pragma unroll
            for (int sg = 0; sg < W; sg++) sym[sg] = sax_symbol(beta, __ddiv_rn(acc[sg], (double)seg));
            const uint64_t id = id0 + r0 + lane;
            uint4 wv;
            wv.x = sym[0] | (sym[1] << 8) | (sym[2] << 16) | (sym[3] << 24);
            wv.y = sym[4] | (sym[5] << 8) | (sym[6] << 16) | (sym[7] << 24);
            wv.z = sym[8] | (sym[9] << 8) | (sym[10] << 16) | (sym[11] << 24);
            wv.w = sym[12] | (sym[13] << 8) | (sym[14] << 16) | (sym[15] << 24);
            reinterpret_cast<uint4 *>(sax_by_id)[id] = wv;
            key[id] = isax_key(sym);
            musig[id] = ms[lane];
            if (!finite) atomicOr(bad, 1u);
        }
        __syncwarp();
    }
}

// Split summarisation for n = 128 and 256: two kernels with no shared-memory staging.
//  moments_kernel: thread per series (mu, sigma: two sequential fp64 chains over the row, read
//    with float4 loads through L1; registers only, so many series are in flight per SM).
//  paa_sax_kernel: a half-warp per series, lane = segment: the lane z-normalises its n/w points
//    (znorm_value, the exact rounding of R3), sums them left to right in fp64 and takes the symbol;
//    the key's bit planes are warp ballots. The per-series operation order is that of
//    summarise_kernel (and of the oracle): identical words.
template <uint32_t NT>
__global__ void __launch_bounds__(256) moments_kernel(const float *__restrict__ x, uint64_t count,
                                                      double2 *__restrict__ ms_out, uint32_t *__restrict__ bad) {
    constexpr uint32_t C = NT / 4, U = 8;  // float4 per row; per group (two groups in flight)
    static_assert(C % (2 * U) == 0, "whole groups");
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < count; r += (uint64_t)gridDim.x * blockDim.x) {
        const float4 *row = reinterpret_cast<const float4 *>(x + r * NT);
        bool finite = true;
        // C1, left to right (R2, R3); the next group's loads are issued before this group's adds
        double s = 0.0;
        float4 a[U], b[U];
#pragma unroll
        for (uint32_t k = 0; k < U; k++) a[k] = __ldg(row + k);
#pragma unroll 1
        for (uint32_t c0 = 0; c0 < C; c0 += 2 * U) {
#pragma unroll
            for (uint32_t k = 0; k < U; k++) b[k] = __ldg(row + c0 + U + k);
#pragma unroll
            for (uint32_t k = 0; k < U; k++) {
                finite &= isfinite(a[k].x) && isfinite(a[k].y) && isfinite(a[k].z) && isfinite(a[k].w);
                s = __dadd_rn(s, (double)(a[k].x));
                s = __dadd_rn(s, (double)(a[k].y));
                s = __dadd_rn(s, (double)(a[k].z));
                s = __dadd_rn(s, (double)(a[k].w));
            }
            if (c0 + 2 * U < C) {
#pragma unroll
                for (uint32_t k = 0; k < U; k++) a[k] = __ldg(row + c0 + 2 * U + k);
            }
#pragma unroll
            for (uint32_t k = 0; k < U; k++) {
                finite &= isfinite(b[k].x) && isfinite(b[k].y) && isfinite(b[k].z) && isfinite(b[k].w);
                s = __dadd_rn(s, (double)(b[k].x));
                s = __dadd_rn(s, (double)(b[k].y));
                s = __dadd_rn(s, (double)(b[k].z));
                s = __dadd_rn(s, (double)(b[k].w));
            }
        }
        const double mu = __ddiv_rn(s, (double)NT);
        double s2 = 0.0;
#pragma unroll
        for (uint32_t k = 0; k < U; k++) a[k] = __ldg(row + k);
#pragma unroll 1
        for (uint32_t c0 = 0; c0 < C; c0 += 2 * U) {
#pragma unroll
            for (uint32_t k = 0; k < U; k++) b[k] = __ldg(row + c0 + U + k);
#pragma unroll
            for (uint32_t k = 0; k < U; k++) {
                double t;
                t = __dsub_rn((double)(a[k].x), mu); s2 = __dadd_rn(s2, __dmul_rn(t, t));
                t = __dsub_rn((double)(a[k].y), mu); s2 = __dadd_rn(s2, __dmul_rn(t, t));
                t = __dsub_rn((double)(a[k].z), mu); s2 = __dadd_rn(s2, __dmul_rn(t, t));
                t = __dsub_rn((double)(a[k].w), mu); s2 = __dadd_rn(s2, __dmul_rn(t, t));
            }
            if (c0 + 2 * U < C) {
#pragma unroll
                for (uint32_t k = 0; k < U; k++) a[k] = __ldg(row + c0 + 2 * U + k);
            }
#pragma unroll
            for (uint32_t k = 0; k < U; k++) {
                double t;
                t = __dsub_rn((double)(b[k].x), mu); s2 = __dadd_rn(s2, __dmul_rn(t, t));
                t = __dsub_rn((double)(b[k].y), mu); s2 = __dadd_rn(s2, __dmul_rn(t, t));
                t = __dsub_rn((double)(b[k].z), mu); s2 = __dadd_rn(s2, __dmul_rn(t, t));
                t = __dsub_rn((double)(b[k].w), mu); s2 = __dadd_rn(s2, __dmul_rn(t, t));
            }
        }
        ms_out[r] = make_double2(mu, __dsqrt_rn(__ddiv_rn(s2, (double)NT)));
        if (!finite) atomicOr(bad, 1u);
    }
}

template <uint32_t NT>
__global__ void __launch_bounds__(256) paa_sax_kernel(const float *__restrict__ x, uint64_t count, uint64_t id0,
                                                      const double2 *__restrict__ musig, uint8_t *__restrict__ sax_by_id,
                                                      uint4 *__restrict__ key) {
    constexpr uint32_t seg = NT / W;
    __shared__ double beta[ISAX_NBETA];
    for (uint32_t k = threadIdx.x; k < ISAX_NBETA; k += blockDim.x) beta[k] = c_beta[k];
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, sg = lane & 15;
    const uint64_t hw0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 4;  // half-warp = one series
    const uint64_t nhw = ((uint64_t)gridDim.x * blockDim.x) >> 4;
    for (uint64_t r0 = hw0 - (hw0 & 1); r0 < count; r0 += nhw) {  // warp-uniform: two series per warp
        const uint64_t r = r0 + (lane >> 4);
        const bool live = r < count;
        uint32_t sym = 0;
        if (live) {
            const double2 m = musig[id0 + r];
            const double rcp = __drcp_rn(m.y);
            const float4 *src = reinterpret_cast<const float4 *>(x + r * NT + sg * seg);
            double acc = 0.0;
#pragma unroll
            for (uint32_t c = 0; c < seg / 4; c++) {
                const float4 v = __ldg(src + c);
                const float y0 = m.y < 1e-12 ? 0.0f : znorm_value(v.x, m.x, m.y, rcp);
                const float y1 = m.y < 1e-12 ? 0.0f : znorm_value(v.y, m.x, m.y, rcp);
                const float y2 = m.y < 1e-12 ? 0.0f : znorm_value(v.z, m.x, m.y, rcp);
                const float y3 = m.y < 1e-12 ? 0.0f : znorm_value(v.w, m.x, m.y, rcp);
                acc = __dadd_rn(acc, (double)y0);
                acc = __dadd_rn(acc, (double)y1);
                acc = __dadd_rn(acc, (double)y2);
                acc = __dadd_rn(acc, (double)y3);
            }
            sym = sax_symbol(beta, __ddiv_rn(acc, (double)seg));
            sax_by_id[(id0 + r) * W + sg] = (uint8_t)sym;
        }
        // key (R6): plane p holds bit (7 - p) of every segment's symbol, segment 0 most significant
        uint32_t plane[8];
#pragma unroll
        for (int p = 0; p < 8; p++) {
            const uint32_t b = __ballot_sync(0xffffffffu, (sym >> (7 - p)) & 1u);
            plane[p] = __brev((lane < 16 ? b : (b >> 16)) & 0xFFFFu) >> 16;
        }
        if (live && sg == 0)
            key[id0 + r] = make_uint4((plane[6] << 16) | plane[7], (plane[4] << 16) | plane[5], (plane[2] << 16) | plane[3],
                                      (plane[0] << 16) | plane[1]);
    }
}

// ------------------------------------------------------------------------------------ TMA tiles
// The default for n = 128 and 256 since round 2c: a CTA of four warps owns a tile of 32 rows. The
// rows arrive by the TMA engine: lane r of warp 0 issues one bulk copy (cp.async.bulk, 4n bytes)
// of row r into its padded shared-memory row, all completing on one mbarrier, so the staging
// costs no registers, no issue slots and no bank-conflicted stores (the round-1 kernel's scalar
// stores were 4-way conflicted, and the split kernels' per-thread global reads cost 32 L1
// wavefronts per warp load). Rows are n + 4 floats apart: a thread reads its row with 16-byte
// loads, and the eight threads of a quarter warp then hit eight different 16-byte bank groups.
// Every sum is strictly left to right with explicit __d*_rn (R3): warp 0, thread = row, takes the
// mean and the variance (two sequential chains); then warp w, lane = row, z-normalises the points
// of segments 4w .. 4w+3 (znorm_value_d: no conversion back and forth) and adds each to its
// segment's sum, four independent chains; symbols by binary search, the key by bit interleave.
// One read of the input from HBM (the split kernels read it twice and converted each point five
// times: here three F2D per point). Six CTAs fit on an SM (36 KB each); a CTA's compute hides the
// other CTAs' copies. The per-series operation order is that of summarise_kernel (and of the
// oracle): identical words.
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t mbar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(mbar), "r"(parity)
        : "memory");
    return ok != 0;
}
// one-dimensional bulk copy global -> shared (the TMA engine; UBLKCP in SASS), completing on mbar
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}

// fp64 value of y = fp32_rne(fl64((x - mu) / sd)) (znorm_value's result, as a double) without the
// two conversions: outside znorm_value's window the low 29 bits of q's significand are not within
// 8 of the halfway point, so rounding to fp32 precision is "add 2^28, clear the low 29 bits" on
// q's bit pattern (a carry moves into the exponent as it should; the exponent range keeps the
// result a normal fp32).
__device__ __forceinline__ double znorm_value_d(float x, double mu, double sd, double rcp) {
    const double t = __dsub_rn((double)x, mu);
    const double q = __dmul_rn(t, rcp);
    const unsigned long long b = (unsigned long long)__double_as_longlong(q);
    const uint32_t ex = (uint32_t)(b >> 52) & 0x7FFu;
    const uint32_t low = (uint32_t)b & ((1u << 29) - 1u);
    if (ex >= 898u && ex <= 1149u && low - ((1u << 28) - 8u) > 16u)
        return __longlong_as_double((long long)((b + (1ull << 28)) & ~((1ull << 29) - 1ull)));
    return (double)__double2float_rn(__ddiv_rn(t, sd));
}

// Four warps per 32-row tile. (One warp per 32-row tile, everything thread = row: 10.2 ms per
// 10M x 256, too few warps per scheduler; one warp per 16-row tile with half-idle lanes in the
// moments: 7.3 ms; this shape: 5.3 ms; the split kernels before it: 8.2 ms.)
#ifndef ISAX_ST_WARPS
#define ISAX_ST_WARPS 4
#endif
constexpr int ST_WARPS = ISAX_ST_WARPS;  // 4 or 8: warp w takes 16 / ST_WARPS segments of every row
constexpr int ST_THREADS = 32 * ST_WARPS;
constexpr int ST_SEGS = W / ST_WARPS;
static_assert(ST_WARPS == 2 || ST_WARPS == 4 || ST_WARPS == 8, "whole segments per warp");
template <uint32_t NT>
__global__ void __launch_bounds__(ST_THREADS) summarise_tma_kernel(const float *__restrict__ x, uint64_t count, uint64_t id0,
                                                                   uint8_t *__restrict__ sax_by_id, uint4 *__restrict__ key,
                                                                   double2 *__restrict__ musig, uint32_t *__restrict__ bad) {
    constexpr uint32_t STRIDE = NT + 4;  // floats between rows
    constexpr uint32_t seg = NT / W;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // [0, 16): the mbarrier | beta | (mu, sigma) [32] | words [32] | rows [32][STRIDE]
    double *beta = reinterpret_cast<double *>(smem_raw + 16);
    constexpr uint32_t MS_OFF = (16 + ISAX_NBETA * 8 + 15) & ~15u;
    double2 *ms = reinterpret_cast<double2 *>(smem_raw + MS_OFF);
    uint8_t *words = smem_raw + MS_OFF + 32 * 16;  // [32 rows][16]
    constexpr uint32_t ROWS_OFF = MS_OFF + 32 * 16 + 32 * 16;
    const float *rows = reinterpret_cast<const float *>(smem_raw + ROWS_OFF);
    const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t rows_sh = mbar + ROWS_OFF;
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (uint32_t k = t; k < ISAX_NBETA; k += ST_THREADS) beta[k] = c_beta[k];
    if (t == 0) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t parity = 0;
    const uint64_t ngroups = (count + 31) / 32;
    for (uint64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const uint64_t r0 = g * 32;
        const uint32_t nrows = (uint32_t)umin64(32, count - r0);
        if (warp == 0) {
            if (lane == 0) mbar_expect_tx(mbar, nrows * NT * 4);
            __syncwarp();
            if (lane < nrows) bulk_g2s(rows_sh + lane * STRIDE * 4, x + (r0 + lane) * NT, NT * 4, mbar);
        }
        const float4 *row4 = reinterpret_cast<const float4 *>(rows + lane * STRIDE);
        // C1 (warp 0, thread = row): mu and sigma, left to right (R2, R3). Only warp 0 waits for the
        // tile; the other warps wait at the barrier below without taking issue slots.
        if (warp == 0) {
            while (!mbar_try_wait(mbar, parity)) {
            }
        }
        parity ^= 1u;
        if (warp == 0 && lane < nrows) {
            bool finite = true;
            double s = 0.0;
#pragma unroll 8
            for (uint32_t c = 0; c < NT / 4; c++) {
                const float4 v = row4[c];
                // (x - x is 0 for a finite x, NaN for NaN or Inf)
                finite &= (v.x - v.x == 0.f) && (v.y - v.y == 0.f) && (v.z - v.z == 0.f) && (v.w - v.w == 0.f);
                s = __dadd_rn(s, (double)v.x);
                s = __dadd_rn(s, (double)v.y);
                s = __dadd_rn(s, (double)v.z);
                s = __dadd_rn(s, (double)v.w);
            }
            const double mu = __ddiv_rn(s, (double)NT);
            double s2 = 0.0;
#pragma unroll 8
            for (uint32_t c = 0; c < NT / 4; c++) {
                const float4 v = row4[c];
                double d;
                d = __dsub_rn((double)v.x, mu); s2 = __dadd_rn(s2, __dmul_rn(d, d));
                d = __dsub_rn((double)v.y, mu); s2 = __dadd_rn(s2, __dmul_rn(d, d));
                d = __dsub_rn((double)v.z, mu); s2 = __dadd_rn(s2, __dmul_rn(d, d));
                d = __dsub_rn((double)v.w, mu); s2 = __dadd_rn(s2, __dmul_rn(d, d));
            }
            ms[lane] = make_double2(mu, __dsqrt_rn(__ddiv_rn(s2, (double)NT)));
            if (!finite) atomicOr(bad, 1u);
        }
        __syncthreads();
        // C2-C4 (warp w, lane = row): segments ST_SEGS w .. ST_SEGS (w + 1) - 1: y = fp32((x - mu) /
        // sigma) as a double and the segment sums, left to right within each segment; then the symbols
        if (lane < nrows) {
            const double2 m = ms[lane];
            const double rcp = __drcp_rn(m.y);
            const bool flat = m.y < 1e-12;
            double acc[ST_SEGS];
#pragma unroll
            for (int k = 0; k < ST_SEGS; k++) acc[k] = 0.0;
#pragma unroll 2
            for (uint32_t c = 0; c < seg / 4; c++) {
#pragma unroll
                for (int k = 0; k < ST_SEGS; k++) {
                    const float4 v = row4[(ST_SEGS * warp + k) * (seg / 4) + c];
                    acc[k] = __dadd_rn(acc[k], flat ? 0.0 : znorm_value_d(v.x, m.x, m.y, rcp));
                    acc[k] = __dadd_rn(acc[k], flat ? 0.0 : znorm_value_d(v.y, m.x, m.y, rcp));
                    acc[k] = __dadd_rn(acc[k], flat ? 0.0 : znorm_value_d(v.z, m.x, m.y, rcp));
                    acc[k] = __dadd_rn(acc[k], flat ? 0.0 : znorm_value_d(v.w, m.x, m.y, rcp));
                }
            }
#pragma unroll
            for (int k = 0; k < ST_SEGS; k++)
                words[lane * W + ST_SEGS * warp + k] = (uint8_t)sax_symbol(beta, __ddiv_rn(acc[k], (double)seg));
        }
        __syncthreads();
        if (warp == 0 && lane < nrows) {
            const uint4 wv = reinterpret_cast<const uint4 *>(words)[lane];
            const uint32_t v[4] = {wv.x, wv.y, wv.z, wv.w};
            uint32_t sym[W];
#pragma unroll
            for (int sg = 0; sg < W; sg++) sym[sg] = (v[sg >> 2] >> (8 * (sg & 3))) & 0xFFu;
            const uint64_t id = id0 + r0 + lane;
            reinterpret_cast<uint4 *>(sax_by_id)[id] = wv;
            key[id] = isax_key(sym);
            musig[id] = ms[lane];
        }
        // the tile's reads (generic proxy) before the next tile's copies (async proxy)
        __syncthreads();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
}

template <uint32_t NT>
static void launch_summarise_tma(const float *x, uint64_t count, uint64_t id0, uint8_t *sax_by_id, uint4 *key,
                                 double2 *musig, uint32_t *bad, cudaStream_t s) {
    const size_t smem = ((16 + ISAX_NBETA * 8 + 15) & ~size_t(15)) + 32 * 16 + 32 * 16 + 32 * (size_t)(NT + 4) * sizeof(float);
    // per launch (the attribute is per device; a failure surfaces as the launch's error)
    cudaFuncSetAttribute(summarise_tma_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(16, (227 * 1024) / (smem + 1024)));
    const uint64_t grid = umin64((count + 31) / 32, (uint64_t)sms * per_sm);
    summarise_tma_kernel<NT><<<(unsigned)grid, ST_THREADS, smem, s>>>(x, count, id0, sax_by_id, key, musig, bad);
}

template <uint32_t NT>
static void launch_summarise_split(const float *x, uint64_t count, uint64_t id0, uint8_t *sax_by_id, uint4 *key,
                                   double2 *musig, uint32_t *bad, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // few series in flight (ISAX_MOM_CTAS CTAs of 256 per SM): the rows being read (1 KB each at
    // n = 256) stay in L2 between the mean and the variance passes
#ifndef ISAX_MOM_CTAS
#define ISAX_MOM_CTAS 2
#endif
    const uint64_t ga = umin64((count + 255) / 256, (uint64_t)sms * ISAX_MOM_CTAS);
    moments_kernel<NT><<<(unsigned)ga, 256, 0, s>>>(x, count, musig + id0, bad);
    const uint64_t gb = umin64((count * 16 + 255) / 256, (uint64_t)sms * 8);
    paa_sax_kernel<NT><<<(unsigned)gb, 256, 0, s>>>(x, count, id0, musig, sax_by_id, key);
}

template <uint32_t NT>
static void launch_summarise_half(const float *x, uint64_t count, uint64_t id0, uint8_t *sax_by_id, uint4 *key,
                                  double2 *musig, uint32_t *bad, cudaStream_t s) {
    const size_t smem = ISAX_NBETA * sizeof(double) + 8 + 32 * sizeof(double2) + 32 * (size_t)(NT / 2 + 1) * sizeof(float);
    static size_t configured = 0;
    if (smem > configured) {
        cudaFuncSetAttribute(summarise_half_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(32, (227 * 1024) / (smem + 1024)));
    const uint64_t grid = umin64((count + 31) / 32, (uint64_t)sms * per_sm);
    summarise_half_kernel<NT><<<(unsigned)grid, 32, smem, s>>>(x, count, id0, sax_by_id, key, musig, bad);
}

template <uint32_t NT>
static void launch_summarise_t(const float *x, uint64_t count, uint32_t n, uint64_t id0, uint8_t *sax_by_id,
                               uint4 *key, double2 *musig, uint32_t *bad, cudaStream_t s) {
    const size_t smem = ISAX_NBETA * sizeof(double) + 8 + 32 * sizeof(double2) + 32 * (size_t)(n + 1) * sizeof(float);
    static size_t configured = 0;
    if (smem > configured) {
        cudaFuncSetAttribute(summarise_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(32, (227 * 1024) / (smem + 1024)));
    const uint64_t groups = (count + 31) / 32;
    const uint64_t grid = umin64(groups, (uint64_t)sms * per_sm);
    summarise_kernel<NT><<<(unsigned)grid, 32, smem, s>>>(x, count, n, id0, sax_by_id, key, musig, bad);
}

void launch_summarise(const float *x, uint64_t count, uint32_t n, uint64_t id0, uint8_t *sax_by_id, uint4 *key,
                      double2 *musig, uint32_t *bad, cudaStream_t s) {
    if (count == 0) return;
#if defined(ISAX_SUMMARISE_HALF)
    if (n == 256) return launch_summarise_half<256>(x, count, id0, sax_by_id, key, musig, bad, s);
    if (n == 128) return launch_summarise_half<128>(x, count, id0, sax_by_id, key, musig, bad, s);
#elif defined(ISAX_SUMMARISE_SPLIT)
    if (n == 256) return launch_summarise_split<256>(x, count, id0, sax_by_id, key, musig, bad, s);
    if (n == 128) return launch_summarise_split<128>(x, count, id0, sax_by_id, key, musig, bad, s);
#elif !defined(ISAX_SUMMARISE_FULLROW)
    // (the bulk copies need 16-byte aligned rows: x from cudaMalloc or a chunk offset of whole rows)
    if (n == 256 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) return launch_summarise_tma<256>(x, count, id0, sax_by_id, key, musig, bad, s);
    if (n == 128 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) return launch_summarise_tma<128>(x, count, id0, sax_by_id, key, musig, bad, s);
#endif
    if (n == 256) launch_summarise_t<256>(x, count, n, id0, sax_by_id, key, musig, bad, s);
    else if (n == 128) launch_summarise_t<128>(x, count, n, id0, sax_by_id, key, musig, bad, s);
    else launch_summarise_t<0>(x, count, n, id0, sax_by_id, key, musig, bad, s);
}

}  // namespace isax
