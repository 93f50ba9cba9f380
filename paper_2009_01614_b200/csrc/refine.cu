// refine.cu: early-abandoning real distances over the candidate lists, then the exact finalise.
//
// "a number of real distance calculation workers consume [the candidate list] in
// parallel and compute the real distances". P:357: "we may find a series with a smaller
// distance to the query, in which case we update the BSF". north_star (b): "refinement with
// early-abandoning squared Euclidean distance and an atomically shrinking BSF".
//
// refine_kernel: one warp per candidate. Candidates from every query of the batch are one
//   flat index space (a prefix over the per-query counts, in shared memory), so a single
//   launch reaches steady state. For each candidate:
//   - it reads the current BSF of its query (relaxed: a stale value is only looser);
//   - it streams the row in 512-byte steps (float4 per lane);
//   - after each step but the last, it abandons iff the partial sum > bsf * (1 + delta) (R8);
//   - on completion it does atomicMin on the packed (d^2, id) word, and appends (id, pos, d^2)
//     to the near list if d^2 <= bsf * (1 + delta) (R9).
// finalize_kernel: one warp per query. Near-list entries within (1 + delta) of the final BSF
//   are recomputed in fp64, in one fixed order for every row. The answer is the
//   lexicographic min of (d^2_fp64, id) (lowest id on ties; north_star). dist = fp32(sqrt(d^2)).
#include "isax_device.cuh"

namespace isax {

constexpr int RF_THREADS = 256;
constexpr int RF_MAXQ = 1024;

template <int NS>
__global__ void __launch_bounds__(RF_THREADS) refine_kernel(const float *__restrict__ stored,
                                                           const uint32_t *__restrict__ perm, uint32_t n,
                                                           const float *__restrict__ qy, uint32_t Q,
                                                           const uint32_t *__restrict__ cand,
                                                           const uint32_t *__restrict__ cand_cnt, uint32_t cap,
                                                           unsigned long long *__restrict__ bsf,
                                                           NearEntry *__restrict__ near, uint32_t *__restrict__ near_cnt,
                                                           uint32_t *__restrict__ counters, float onepd) {
    __shared__ uint32_t pre[RF_MAXQ + 1];
    const uint32_t t = threadIdx.x, lane = t & 31;
    if (t == 0) {
        uint32_t run = 0;
        for (uint32_t q = 0; q < Q; q++) {
            pre[q] = run;
            run += cand_cnt[q] <= cap ? cand_cnt[q] : 0;  // an overflowed list is redone (cand_prefix)
        }
        pre[Q] = run;
    }
    __syncthreads();
    const uint32_t total = pre[Q];
    const uint32_t nwarps = gridDim.x * (RF_THREADS / 32);
    uint32_t cur_q = 0xffffffffu;
    float4 qv[NS];
    uint32_t done = 0, abandoned = 0;
    for (uint32_t f = blockIdx.x * (RF_THREADS / 32) + (t >> 5); f < total; f += nwarps) {
        uint32_t lo = 0, hi = Q;  // last q with pre[q] <= f
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (pre[mid] <= f) lo = mid;
            else hi = mid;
        }
        const uint32_t q = lo;
        if (q != cur_q) {
            if (cur_q != 0xffffffffu && lane == 0) {
                atomicAdd(&counters[4 * cur_q + 0], done);
                atomicAdd(&counters[4 * cur_q + 1], abandoned);
            }
            done = abandoned = 0;
            cur_q = q;
#pragma unroll
            for (int k = 0; k < NS; k++) {
                const uint32_t i = k * 128 + 4 * lane;
                qv[k] = i < n ? *reinterpret_cast<const float4 *>(qy + (uint64_t)q * n + i) : make_float4(0, 0, 0, 0);
            }
        }
        const uint32_t pos = cand[(uint64_t)q * cap + (f - pre[q])];
        const float *row = stored + (uint64_t)pos * n;
        const float lim = bsf_d2(*((volatile unsigned long long *)&bsf[q])) * onepd;
        float acc = 0.f;
        bool ab = false;
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
            if (k + 1 < NS && (k + 1) * 128 < n) {
                if (warp_sum(acc) > lim) {  // early abandon (R8)
                    ab = true;
                    break;
                }
            }
        }
        if (ab) {
            abandoned++;
            continue;
        }
        const float d2 = warp_sum(acc);
        done++;
        if (lane == 0 && d2 <= lim) {
            const uint32_t id = perm[pos];
            atomicMin(&bsf[q], pack_bsf(d2, id));
            const uint32_t k = atomicAdd(&near_cnt[q], 1u);
            if (k < NEAR_K) near[(uint64_t)q * NEAR_K + k] = NearEntry{id, pos, d2, 0};
        }
    }
    if (cur_q != 0xffffffffu && lane == 0) {
        atomicAdd(&counters[4 * cur_q + 0], done);
        atomicAdd(&counters[4 * cur_q + 1], abandoned);
    }
}

// Quarter-warp variant for n <= 256 (the paper's lengths, 128 and 256). Eight lanes own a
// candidate and keep two candidates in flight: both first halves are loaded before either is
// reduced, which gives each lane 2 NH float4 outstanding. At n = 256 that is 1 KB per quarter
// and 4 KB per warp. The abandon check after the first half reduces over the quarter's 8 lanes
// (3 xor shuffles). The query row is read through the read-only path (L1-resident).
// The BSF threshold is refreshed from L2 every RF_REFRESH candidates; a stale value is only
// looser. Same arithmetic contract as refine_kernel.
constexpr uint32_t RF_REFRESH = 4;
#ifndef ISAX_RF_C
#define ISAX_RF_C 2
#endif
constexpr int RF_C = ISAX_RF_C;  // candidates in flight per quarter warp

template <int NH>
__global__ void __launch_bounds__(RF_THREADS) refine_q_kernel(const float *__restrict__ stored,
                                                             const uint32_t *__restrict__ perm, uint32_t n,
                                                             const float *__restrict__ qy, uint32_t Q,
                                                             const uint32_t *__restrict__ cand,
                                                             const uint8_t *__restrict__ candq,
                                                             const float *__restrict__ qscale,
                                                             const uint32_t *__restrict__ cand_cnt, uint32_t cap,
                                                             unsigned long long *__restrict__ bsf,
                                                             NearEntry *__restrict__ near,
                                                             uint32_t *__restrict__ near_cnt,
                                                             uint32_t *__restrict__ counters, float onepd,
                                                             unsigned long long *__restrict__ refine_bytes) {
    __shared__ uint32_t pre[RF_MAXQ + 1];
    const uint32_t t = threadIdx.x, lane = t & 31, ql = lane & 7;
    unsigned long long rows_read = 0;  // half rows read by this quarter
    const uint32_t qmask = 0xFFu << (lane & 24);
    cand_prefix<RF_THREADS>(cand_cnt, Q, cap, pre);
    const uint32_t total = pre[Q];
    const uint32_t nquart = gridDim.x * (RF_THREADS / 8);
    auto locate = [&](uint32_t f) {  // last q with pre[q] <= f
        uint32_t lo = 0, hi = Q;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (pre[mid] <= f) lo = mid;
            else hi = mid;
        }
        return lo;
    };
    uint32_t cur_q = 0xffffffffu, done = 0, abandoned = 0, since = 0;
    float lim_c = 0.f;
    // each quarter owns a contiguous range of the flat candidate index: consecutive candidates
    // share a query (its counters are flushed only when the query changes) and sit close together
    // in the sorted order
    const uint32_t per = (total + nquart - 1) / nquart;
    const uint32_t qi = (blockIdx.x * RF_THREADS + t) >> 3;
    const uint32_t fbeg = min(qi * per, total), fend = min(fbeg + per, total);
    for (uint32_t f0 = fbeg; f0 < fend; f0 += RF_C) {
        uint32_t qv[RF_C], pv[RF_C];
        bool live[RF_C];
#pragma unroll
        for (int c = 0; c < RF_C; c++) {
            const uint32_t f = f0 + c;
            live[c] = f < fend;
            qv[c] = live[c] ? locate(f) : 0;
            pv[c] = live[c] ? cand[(uint64_t)qv[c] * cap + (f - pre[qv[c]])] : 0;
        }
        float4 v[RF_C][NH];
#pragma unroll
        for (int c = 0; c < RF_C; c++)
#pragma unroll
            for (int k = 0; k < NH; k++)
                v[c][k] = live[c] ? __ldcs(reinterpret_cast<const float4 *>(stored + (uint64_t)pv[c] * n) + k * 8 + ql)
                                  : make_float4(0, 0, 0, 0);
#pragma unroll
        for (int c = 0; c < RF_C; c++) {
            if (!live[c]) continue;
            const uint32_t q = qv[c], pos = pv[c];
            if (q != cur_q) {
                if (cur_q != 0xffffffffu && ql == 0) {
                    atomicAdd(&counters[4 * cur_q + 0], done);
                    atomicAdd(&counters[4 * cur_q + 1], abandoned);
                }
                rows_read += 2 * done + abandoned;
                done = abandoned = 0;
                cur_q = q;
                since = RF_REFRESH;
            }
            if (since++ >= RF_REFRESH) {
                // read by the quarter's first lane and broadcast: the quarter's lanes must take the
                // same abandon decision (their shuffles below assume it)
                float l = 0.f;
                if (ql == 0) l = bsf_d2(*((volatile unsigned long long *)&bsf[q])) * onepd;
                lim_c = __shfl_sync(qmask, l, lane & 24);
                since = 1;
            }
            const float lim = lim_c;
            const float4 *qr = reinterpret_cast<const float4 *>(qy + (uint64_t)q * n);
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < NH; k++) {
                const float4 w = __ldg(qr + k * 8 + ql);
                float d;
                d = v[c][k].x - w.x; acc = fmaf(d, d, acc);
                d = v[c][k].y - w.y; acc = fmaf(d, d, acc);
                d = v[c][k].z - w.z; acc = fmaf(d, d, acc);
                d = v[c][k].w - w.w; acc = fmaf(d, d, acc);
            }
            float part = acc;
            part += __shfl_xor_sync(qmask, part, 1);
            part += __shfl_xor_sync(qmask, part, 2);
            part += __shfl_xor_sync(qmask, part, 4);
            if (part > lim) {  // early abandon after half the row (R8)
                abandoned++;
                continue;
            }
            const float4 *row = reinterpret_cast<const float4 *>(stored + (uint64_t)pos * n);
            float4 u[NH];
#pragma unroll
            for (int k = 0; k < NH; k++) u[k] = __ldcs(row + 8 * NH + k * 8 + ql);
#pragma unroll
            for (int k = 0; k < NH; k++) {
                const float4 w = __ldg(qr + 8 * NH + k * 8 + ql);
                float d;
                d = u[k].x - w.x; acc = fmaf(d, d, acc);
                d = u[k].y - w.y; acc = fmaf(d, d, acc);
                d = u[k].z - w.z; acc = fmaf(d, d, acc);
                d = u[k].w - w.w; acc = fmaf(d, d, acc);
            }
            acc += __shfl_xor_sync(qmask, acc, 1);
            acc += __shfl_xor_sync(qmask, acc, 2);
            acc += __shfl_xor_sync(qmask, acc, 4);
            done++;
            if (acc <= lim) {
                // re-read the current BSF before claiming a near slot (the cached one may be stale)
                float cur = 0.f;
                if (ql == 0) cur = bsf_d2(*((volatile unsigned long long *)&bsf[q])) * onepd;
                cur = __shfl_sync(qmask, cur, lane & 24);
                lim_c = cur;
                if (ql == 0 && acc <= cur) {
                    const uint32_t id = perm[pos];
                    atomicMin(&bsf[q], pack_bsf(acc, id));
                    const uint32_t k = atomicAdd(&near_cnt[q], 1u);
                    if (k < NEAR_K) near[(uint64_t)q * NEAR_K + k] = NearEntry{id, pos, acc, 0};
                }
            }
        }
    }
    if (cur_q != 0xffffffffu && ql == 0) {
        atomicAdd(&counters[4 * cur_q + 0], done);
        atomicAdd(&counters[4 * cur_q + 1], abandoned);
    }
    rows_read += 2 * done + abandoned;
    if (ql == 0 && rows_read) atomicAdd(refine_bytes, rows_read * 2ull * n);
}

// The second refine pass's list (MESSI's priority order, approximated by two bands):
// candcheck_kernel puts a large query's candidates with b > B_SPLIT (LB^2 above about 0.55 T) at
// the back of its cand2 region. After the first pass has tightened the BSF, filter_kernel keeps of
// them only those that pass the skip test (R11b): b / sc <= LB^2, so b > lim * sc (rounded up)
// means LB^2 > lim = bsf^2 (1 + delta), and the row can hold neither a new answer nor a near tie.
// The survivors go to the front of the scan's own list (cand, free again) for the second pass.
__global__ void __launch_bounds__(RF_THREADS) filter_kernel(const uint32_t *__restrict__ cand2,
                                                           const uint8_t *__restrict__ candq2,
                                                           const uint32_t *__restrict__ cnt_hi, uint32_t Q, uint32_t cap,
                                                           const unsigned long long *__restrict__ bsf,
                                                           const float *__restrict__ qscale, float onepd,
                                                           uint32_t *__restrict__ out, uint32_t *__restrict__ cnt_f,
                                                           uint32_t *__restrict__ counters) {
    constexpr int U = 8;  // candidates per thread per iteration, loads in flight together
    __shared__ uint32_t pre[RF_MAXQ + 1];
    constexpr uint32_t FULL = 0xffffffffu;
    const uint32_t t = threadIdx.x, lane = t & 31;
    const uint32_t lt = (1u << lane) - 1u;
    cand_prefix<RF_THREADS>(cnt_hi, Q, cap, pre);
    const uint32_t total = pre[Q];
    // one contiguous slice per CTA (its queries change rarely)
    const uint32_t per = (total + gridDim.x - 1) / gridDim.x;
    const uint32_t f0 = min(blockIdx.x * per, total), f1 = min(f0 + per, total);
    if (f0 >= f1) return;
    uint32_t q = 0;
    {
        uint32_t lo = 0, hi = Q;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (pre[mid] <= f0) lo = mid;
            else hi = mid;
        }
        q = lo;
    }
    for (uint32_t fb = f0; fb < f1; fb += U * RF_THREADS) {
        uint32_t qk[U], pos[U];
        bool valid[U], live[U];
        float thr[U];
        bool one_q = true;
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t f = fb + u * RF_THREADS + t;
            valid[u] = f < f1;
            if (valid[u])
                while (pre[q + 1] <= f) q++;
            qk[u] = q;
            one_q &= !valid[u] || q == qk[0];
            const uint64_t k = (uint64_t)q * cap + (cap - 1 - (f - pre[q]));
            pos[u] = valid[u] ? cand2[k] : 0u;
            thr[u] = valid[u] ? (float)candq2[k] : 0.f;
        }
        // the skip test against the BSF as it stands now (read once per lane)
        const float lim = bsf_d2(*((volatile const unsigned long long *)&bsf[qk[0]])) * onepd;
        const float scq = qscale[qk[0]];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const float l = qk[u] == qk[0] ? lim : bsf_d2(*((volatile const unsigned long long *)&bsf[qk[u]])) * onepd;
            const float sc = qk[u] == qk[0] ? scq : qscale[qk[u]];
            live[u] = valid[u] && !(thr[u] > __fmul_ru(l, sc));
        }
        const uint32_t q_w = __shfl_sync(FULL, qk[0], 0);  // (every lane shuffles: no short circuit)
        if (__all_sync(FULL, one_q && qk[0] == q_w)) {
            uint32_t bl[U], cl = 0, cs = 0;
#pragma unroll
            for (int u = 0; u < U; u++) {
                bl[u] = __ballot_sync(FULL, live[u]);
                cl += __popc(bl[u]);
                cs += __popc(__ballot_sync(FULL, valid[u] && !live[u]));
            }
            uint32_t base = 0;
            if (lane == 0 && cl) base = atomicAdd(&cnt_f[q_w], cl);
            if (lane == 1 && cs) atomicAdd(&counters[4 * q_w + 2], cs);
            base = __shfl_sync(FULL, base, 0);
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (live[u]) out[(uint64_t)q_w * cap + base + __popc(bl[u] & lt)] = pos[u];
                base += __popc(bl[u]);
            }
        } else {
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t peers = __match_any_sync(FULL, valid[u] ? 2 * qk[u] + (live[u] ? 1u : 0u) : 0xffffffffu);
                if (valid[u]) {
                    const uint32_t leader = __ffs(peers) - 1;
                    uint32_t base = 0;
                    if (lane == leader)
                        base = atomicAdd(live[u] ? &cnt_f[qk[u]] : &counters[4 * qk[u] + 2], (uint32_t)__popc(peers));
                    base = __shfl_sync(peers, base, leader);
                    if (live[u]) out[(uint64_t)qk[u] * cap + base + __popc(peers & lt)] = pos[u];
                }
            }
        }
    }
}

void launch_refine(const isax_index *ix, uint32_t Q, float delta, cudaStream_t s) {
    const QueryScratch &qs = ix->qs;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const float onepd = 1.0f + delta;
    // pass 1: cand2[q][0 .. cand_cnt2); then the filtered second band into cand[q][0 .. cnt_f)
    auto pass = [&](const uint32_t *list, const uint32_t *cnt) {
        if (ix->n <= 256) {
            int per_sm = 1;
            const uint32_t nh = ix->n / 64;
            if (nh == 4) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, refine_q_kernel<4>, RF_THREADS, 0);
            else if (nh == 2) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, refine_q_kernel<2>, RF_THREADS, 0);
            else per_sm = 4;
            const unsigned grid = sms * std::max(1, per_sm);  // exactly one full wave
            switch (nh) {
#define RQ_CASE(K)                                                                                                  \
    case K:                                                                                                         \
        refine_q_kernel<K><<<grid, RF_THREADS, 0, s>>>(ix->stored, ix->perm, ix->n, qs.qy, Q, list, nullptr, nullptr, \
                                                       cnt, qs.cand_cap, qs.bsf, qs.near, qs.near_cnt, qs.counters, \
                                                       onepd, qs.refine_bytes);                                     \
        break;
                RQ_CASE(1) RQ_CASE(2) RQ_CASE(3) RQ_CASE(4)
#undef RQ_CASE
            }
            return;
        }
        const unsigned grid = sms * 8;
        const uint32_t ns = (ix->n + 127) / 128;
#define RF_CASE(K)                                                                                              \
    case K:                                                                                                     \
        refine_kernel<K><<<grid, RF_THREADS, 0, s>>>(ix->stored, ix->perm, ix->n, qs.qy, Q, list, cnt,            \
                                                     qs.cand_cap, qs.bsf, qs.near, qs.near_cnt, qs.counters, onepd); \
        break;
        switch (ns) {
            RF_CASE(1) RF_CASE(2) RF_CASE(3) RF_CASE(4) RF_CASE(5) RF_CASE(6) RF_CASE(7) RF_CASE(8)
        }
#undef RF_CASE
    };
    pass(qs.cand2, qs.cand_cnt2);
    filter_kernel<<<sms * 4, RF_THREADS, 0, s>>>(qs.cand2, qs.candq2, qs.cnt_hi, Q, qs.cand_cap, qs.bsf, qs.qscale,
                                                 onepd, qs.cand, qs.cnt_f, qs.counters);
    pass(qs.cand, qs.cnt_f);
}

// ------------------------------------------------------------------------------------ finalize
__global__ void __launch_bounds__(32) finalize_kernel(const float *__restrict__ stored, uint32_t n,
                                                      const float *__restrict__ qy,
                                                      const unsigned long long *__restrict__ bsf,
                                                      const NearEntry *__restrict__ near,
                                                      const uint32_t *__restrict__ near_cnt, float onepd,
                                                      int64_t *__restrict__ out_id, float *__restrict__ out_dist) {
    const uint32_t q = blockIdx.x, lane = threadIdx.x;
    const unsigned long long fin = bsf[q];
    const float lim = bsf_d2(fin) * onepd;
    const uint32_t cnt = min(near_cnt[q], (uint32_t)NEAR_K);
    double best = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    uint32_t best_id = (uint32_t)(fin & 0xffffffffu);
    bool have = false;
    for (uint32_t k = 0; k < cnt; k++) {
        const NearEntry e = near[(uint64_t)q * NEAR_K + k];
        if (!(e.d2 <= lim)) continue;
        const float *row = stored + (uint64_t)e.pos * n;
        const float *qr = qy + (uint64_t)q * n;
        double acc = 0.0;
        for (uint32_t i = lane; i < n; i += 32) {
            const double d = __dsub_rn((double)qr[i], (double)row[i]);
            acc = __dadd_rn(acc, __dmul_rn(d, d));
        }
        acc = warp_sum_d(acc);
        if (!have || acc < best || (acc == best && e.id < best_id)) {
            best = acc;
            best_id = e.id;
            have = true;
        }
    }
    if (lane == 0) {
        out_id[q] = (int64_t)best_id;
        out_dist[q] = have ? __double2float_rn(sqrt(best)) : sqrtf(bsf_d2(fin));
    }
}

void launch_finalize(const isax_index *ix, uint32_t Q, float delta, int64_t *out_id, float *out_dist,
                     cudaStream_t s) {
    const QueryScratch &qs = ix->qs;
    finalize_kernel<<<Q, 32, 0, s>>>(ix->stored, ix->n, qs.qy, qs.bsf, qs.near, qs.near_cnt, 1.0f + delta, out_id,
                                     out_dist);
}

}  // namespace isax
