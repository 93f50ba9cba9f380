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
// finalize_kernel: one CTA per query. Near-list entries within (1 + delta) of the final BSF are
//   screened in fp64 and the possible answers compared exactly (integer d^2). The answer is the
//   lexicographic min of (exact d^2, id) (lowest id on ties; north_star). dist = fp32(sqrt(d^2_fp64)).
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
                                                           unsigned long long *__restrict__ bsf, NearList nl,
                                                           uint32_t *__restrict__ counters, float onepd, uint32_t N) {
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
        ISAX_BOUND(pos < N && f - pre[q] < cap);
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
            near_append(nl, q, id, pos, d2);
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
                                                             const uint16_t *__restrict__ candq,
                                                             const float *__restrict__ qscale,
                                                             const uint32_t *__restrict__ cand_cnt, uint32_t cap,
                                                             unsigned long long *__restrict__ bsf, NearList nl,
                                                             uint32_t *__restrict__ counters, float onepd,
                                                             unsigned long long *__restrict__ refine_bytes, uint32_t N) {
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
    uint32_t cur_q = 0xffffffffu, done = 0, abandoned = 0, since = 0, q_rc = 0xffffffffu;
    float lim_c = 0.f, rsc = 0.f;
    // each quarter owns a contiguous range of the flat candidate index: consecutive candidates
    // share a query (its counters are flushed only when the query changes) and sit close together
    // in the sorted order
    const uint32_t per = (total + nquart - 1) / nquart;
    const uint32_t qi = (blockIdx.x * RF_THREADS + t) >> 3;
    const uint32_t fbeg = min(qi * per, total), fend = min(fbeg + per, total);
    // The next step's candidates (query, position, second-half bound) are fetched while this
    // step's rows load, so the list read is off the row loads' dependency chain. The query of
    // f advances from the previous one (the range is contiguous).
    uint32_t qh = fbeg < fend ? locate(fbeg) : 0;
    uint32_t qn[RF_C], pn[RF_C], bn[RF_C];
    auto fetch = [&](uint32_t f0) {
#pragma unroll
        for (int c = 0; c < RF_C; c++) {
            const uint32_t f = f0 + c;
            const bool l = f < fend;
            if (l)
                while (pre[qh + 1] <= f) qh++;
            qn[c] = qh;
            const uint64_t k = (uint64_t)qh * cap + (f - pre[qh]);
            pn[c] = l ? cand[k] : 0xffffffffu;
            bn[c] = l && candq ? (uint32_t)(candq[k] >> 8) : 0u;
        }
    };
    fetch(fbeg);
    for (uint32_t f0 = fbeg; f0 < fend; f0 += RF_C) {
        uint32_t qv[RF_C], pv[RF_C], b2v[RF_C];
        bool live[RF_C];
#pragma unroll
        for (int c = 0; c < RF_C; c++) {
            live[c] = f0 + c < fend;
            qv[c] = qn[c];
            pv[c] = pn[c];
            ISAX_BOUND(!live[c] || (pv[c] < N && qv[c] < Q));
            b2v[c] = bn[c];
        }
        float4 v[RF_C][NH];
#pragma unroll
        for (int c = 0; c < RF_C; c++)
#pragma unroll
            for (int k = 0; k < NH; k++)
                v[c][k] = live[c] ? __ldcs(reinterpret_cast<const float4 *>(stored + (uint64_t)pv[c] * n) + k * 8 + ql)
                                  : make_float4(0, 0, 0, 0);
        if (f0 + RF_C < fend) fetch(f0 + RF_C);
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
            if (q != q_rc) {  // 1 / sc of the query's scan, rounded down (R16)
                q_rc = q;
                rsc = qscale ? __frcp_rd(__ldg(qscale + q)) : 0.f;
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
            // early abandon after half the row (R8): the partial sum plus a lower bound of
            // the second half's distance, b2 / sc <= LB^2 of segments 8..15 <= its ED^2 (R16)
            if (part + __fmul_rd((float)b2v[c], rsc) > lim) {
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
                    near_append(nl, q, id, pos, acc);
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
                                                           const uint16_t *__restrict__ candq2,
                                                           const uint32_t *__restrict__ cnt_hi, uint32_t Q, uint32_t cap,
                                                           const unsigned long long *__restrict__ bsf,
                                                           const float *__restrict__ qscale, float onepd,
                                                           uint32_t *__restrict__ out, uint16_t *__restrict__ outq,
                                                           uint32_t *__restrict__ cnt_f, uint32_t *__restrict__ counters) {
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
        uint32_t qk[U], pos[U], bq[U];
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
            bq[u] = valid[u] ? candq2[k] : 0u;
            thr[u] = (float)(bq[u] & 0xFFu);
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
                if (live[u]) {
                    const uint64_t k = (uint64_t)q_w * cap + base + __popc(bl[u] & lt);
                    out[k] = pos[u];
                    outq[k] = (uint16_t)bq[u];
                }
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
                    if (live[u]) {
                        const uint64_t k = (uint64_t)qk[u] * cap + base + __popc(peers & lt);
                        out[k] = pos[u];
                        outq[k] = (uint16_t)bq[u];
                    }
                }
            }
        }
    }
}

void launch_refine(const isax_index *ix, uint32_t Q, float delta, cudaStream_t s, cudaEvent_t *evs) {
    const QueryScratch &qs = ix->qs;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const float onepd = 1.0f + delta;
    const NearList nl{qs.near, qs.near_off, qs.near_cap, qs.near_cnt};
    // pass 1: cand2[q][0 .. cand_cnt2); then the filtered second band into cand[q][0 .. cnt_f)
    auto pass = [&](const uint32_t *list, const uint16_t *listq, const uint32_t *cnt, unsigned long long *bytes) {
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
        refine_q_kernel<K><<<grid, RF_THREADS, 0, s>>>(ix->stored, ix->perm, ix->n, qs.qy, Q, list, listq, qs.qscale, \
                                                       cnt, qs.cand_cap, qs.bsf, nl, qs.counters,                   \
                                                       onepd, bytes, (uint32_t)ix->N);                              \
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
                                                     qs.cand_cap, qs.bsf, nl, qs.counters, onepd, (uint32_t)ix->N);  \
        break;
        switch (ns) {
            RF_CASE(1) RF_CASE(2) RF_CASE(3) RF_CASE(4) RF_CASE(5) RF_CASE(6) RF_CASE(7) RF_CASE(8)
        }
#undef RF_CASE
    };
    pass(qs.cand2, qs.candq2, qs.cand_cnt2, qs.refine_bytes);
    if (evs) cudaEventRecord(evs[0], s);
    filter_kernel<<<sms * 4, RF_THREADS, 0, s>>>(qs.cand2, qs.candq2, qs.cnt_hi, Q, qs.cand_cap, qs.bsf, qs.qscale,
                                                 onepd, qs.cand, qs.candq, qs.cnt_f, qs.counters);
    if (evs) cudaEventRecord(evs[1], s);
    pass(qs.cand, qs.candq, qs.cnt_f, qs.refine_bytes + 1);
}

// ------------------------------------------------------------------------------------ finalize
// R9: the answer is the lexicographic minimum of (exact d^2, id) over the rows whose fp32 d^2 is
// within (1 + delta) of the final BSF. Every such row is in the query's near list (its partial
// sums never pass the threshold, so it completes, and it is appended when it completes).
//
// One CTA per scanned query. Pass 1 computes d^2 in fp64 for each listed row (differences and
// squares rounded once each, sum in a fixed lane order) and its minimum m64. Every term is >= 0,
// so the fp64 sum is within gamma = (n + 3) 2^-53 (< 1.2e-13 at n <= 1024) of the exact d^2,
// relatively; a row whose exact d^2 is the minimum has fp64 d^2 <= m64 (1 + gamma) / (1 - gamma),
// so the rows with fp64 d^2 <= m64 (1 + 4e-13) are the only possible answers ("eligible").
// Pass 2 finds the lowest and highest id among the eligible rows; if they are equal (the usual
// case: one row, possibly listed twice), that row is the answer. Otherwise pass 3 evaluates d^2
// of every eligible row exactly, as an integer (below), and takes the lexicographic minimum.
// The fp64 values of the first 512 entries are kept in shared memory between the passes.
//
// Exact d^2. A finite fp32 value v is an integer multiple of 2^-149: v = +-M 2^(sh - 149) with M
// the 24-bit significand (23 bits for subnormals, sh = 0) and sh = biased exponent - 1. So
// A = v 2^149 = +-M << sh is an integer, d = A - B is exact, and sum d^2 = 2^298 d^2(v, w) is an
// exact integer too. The stored rows and the query are z-normalised (sum y^2 = n <= 1024, so
// |y| <= 32 < 2^18): A < 2^(24 + 167) fits in six 32-bit limbs, d^2 in twelve. Each lane squares
// its elements' differences into carry-save accumulators (u64 per 32-bit limb position: at most
// 12 additions of < 2^32 per term, 32 terms per lane, 32 lanes: < 2^46, no overflow), the warp
// adds them, and one lane propagates the carries. Keys compare from the top limb down.
constexpr int FZ_THREADS = 256;
constexpr int XL = 6;        // 32-bit limbs of |A - B|
constexpr int XK = 2 * XL;   // limbs of the squared sum

__device__ __forceinline__ void fp32_fixed(float v, uint32_t &neg, uint32_t (&a)[XL]) {
    const uint32_t u = __float_as_uint(v);
    const uint32_t e = (u >> 23) & 0xFFu, mant = u & 0x7FFFFFu;
    const uint32_t M = e ? (mant | 0x800000u) : mant;
    const uint32_t sh = e ? e - 1u : 0u;
    const unsigned long long w = (unsigned long long)M << (sh & 31u);
    const uint32_t j = sh >> 5;
    neg = u >> 31;
#pragma unroll
    for (int i = 0; i < XL; i++) a[i] = (uint32_t)i == j ? (uint32_t)w : ((uint32_t)i == j + 1 ? (uint32_t)(w >> 32) : 0u);
}

// acc += (a - b)^2, exactly (carry-save, base 2^32)
__device__ __forceinline__ void exact_term(float av, float bv, unsigned long long (&acc)[XK + 1]) {
    uint32_t na, nb, a[XL], b[XL], x[XL];
    fp32_fixed(av, na, a);
    fp32_fixed(bv, nb, b);
    if (na != nb) {  // |a - b| = |a| + |b|
        unsigned long long c = 0;
#pragma unroll
        for (int i = 0; i < XL; i++) {
            c += (unsigned long long)a[i] + b[i];
            x[i] = (uint32_t)c;
            c >>= 32;
        }
    } else {  // |a - b| = | |a| - |b| |
        long long br = 0;
#pragma unroll
        for (int i = 0; i < XL; i++) {
            const long long t = (long long)a[i] - (long long)b[i] + br;
            x[i] = (uint32_t)t;
            br = t >> 32;  // 0 or -1
        }
        if (br) {  // negative: two's complement
            unsigned long long c = 1;
#pragma unroll
            for (int i = 0; i < XL; i++) {
                c += (unsigned long long)(~x[i]);
                x[i] = (uint32_t)c;
                c >>= 32;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < XL; i++)
#pragma unroll
        for (int j = 0; j < XL; j++) {
            const unsigned long long p = (unsigned long long)x[i] * x[j];
            acc[i + j] += (uint32_t)p;
            acc[i + j + 1] += p >> 32;
        }
}

// exact key of one listed row (its XK limbs, most significant last), computed by one warp
__device__ __forceinline__ void exact_key(const float *__restrict__ row, const float *__restrict__ qr, uint32_t n,
                                          uint32_t lane, uint32_t (&key)[XK]) {
    unsigned long long acc[XK + 1];
#pragma unroll
    for (int i = 0; i <= XK; i++) acc[i] = 0;
    for (uint32_t i = lane; i < n; i += 32) exact_term(qr[i], row[i], acc);
#pragma unroll
    for (int i = 0; i <= XK; i++)
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
    unsigned long long c = 0;
#pragma unroll
    for (int i = 0; i < XK; i++) {
        c += acc[i];
        key[i] = (uint32_t)c;
        c >>= 32;
    }
}

__device__ __forceinline__ bool key_id_less(const uint32_t (&a)[XK], uint32_t ida, const uint32_t (&b)[XK], uint32_t idb) {
#pragma unroll
    for (int i = XK - 1; i >= 0; i--)
        if (a[i] != b[i]) return a[i] < b[i];
    return ida < idb;
}

__device__ __forceinline__ double row_d64(const float *__restrict__ row, const float *__restrict__ qr, uint32_t n,
                                          uint32_t lane) {
    double acc = 0.0;
    for (uint32_t i = lane; i < n; i += 32) {
        const double d = __dsub_rn((double)qr[i], (double)row[i]);
        acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
    return warp_sum_d(acc);
}

__global__ void __launch_bounds__(FZ_THREADS) finalize_kernel(const float *__restrict__ stored, uint32_t n,
                                                              const float *__restrict__ qy, const uint32_t *__restrict__ qmap,
                                                              const unsigned long long *__restrict__ bsf, NearList nl,
                                                              float onepd, int64_t *__restrict__ out_id,
                                                              float *__restrict__ out_dist) {
    constexpr uint32_t NWF = FZ_THREADS / 32;
    constexpr uint32_t CACHE = 512;  // fp64 d^2 of the first entries, kept between the passes
    __shared__ double s_dv[CACHE];
    __shared__ double s_m[NWF];
    __shared__ uint32_t s_lo[NWF], s_hi[NWF], s_pos[NWF];
    __shared__ uint32_t s_key[NWF][XK];
    __shared__ uint32_t s_id[NWF];
    __shared__ double s_d64[NWF];
    const uint32_t q = qmap[blockIdx.x];
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const unsigned long long fin = bsf[q];
    const float lim = bsf_d2(fin) * onepd;
    const uint32_t cnt = min(nl.cnt[q], nl.cap[q]);
    const NearEntry *list = nl.base + nl.off[q];
    ISAX_BOUND(cnt <= nl.cap[q]);
    const float *qr = qy + (uint64_t)q * n;
    const double INF64 = __longlong_as_double(0x7ff0000000000000ll);
    // fp64 d^2 of entry k (+inf if it is not within (1 + delta) of the final BSF)
    auto d64_of = [&](uint32_t k, const NearEntry &e) -> double {
        if (k < CACHE) return s_dv[k];
        return e.d2 <= lim ? row_d64(stored + (uint64_t)e.pos * n, qr, n, lane) : INF64;
    };
    // pass 1: fp64 d^2 of every listed row and their minimum
    double m = INF64;
    for (uint32_t k = warp; k < cnt; k += NWF) {
        const NearEntry e = list[k];
        const double d = e.d2 <= lim ? row_d64(stored + (uint64_t)e.pos * n, qr, n, lane) : INF64;
        if (k < CACHE && lane == 0) s_dv[k] = d;
        m = fmin(m, d);
    }
    if (lane == 0) s_m[warp] = m;
    __syncthreads();
    m = INF64;
    for (uint32_t w = 0; w < NWF; w++) m = fmin(m, s_m[w]);
    if (m == INF64) {  // nothing listed (unreachable: the BSF's own row is listed); the BSF word's id
        if (t == 0) {
            out_id[q] = (int64_t)(uint32_t)(fin & 0xffffffffu);
            out_dist[q] = sqrtf(bsf_d2(fin));
        }
        return;
    }
    const double elig = m * (1.0 + 4e-13);
    // pass 2: the lowest and highest id among the eligible rows
    uint32_t lo_id = 0xffffffffu, hi_id = 0, lo_pos = 0;
    for (uint32_t k = warp; k < cnt; k += NWF) {
        const NearEntry e = list[k];
        if (d64_of(k, e) <= elig) {
            if (e.id < lo_id) {
                lo_id = e.id;
                lo_pos = e.pos;
            }
            hi_id = max(hi_id, e.id);
        }
    }
    if (lane == 0) {
        s_lo[warp] = lo_id;
        s_hi[warp] = hi_id;
        s_pos[warp] = lo_pos;
    }
    __syncthreads();
    for (uint32_t w = 0; w < NWF; w++) {
        if (s_lo[w] < lo_id) {
            lo_id = s_lo[w];
            lo_pos = s_pos[w];
        }
        hi_id = max(hi_id, s_hi[w]);
    }
    if (lo_id == hi_id) {  // one eligible row (possibly listed more than once): the answer
        const double d = row_d64(stored + (uint64_t)lo_pos * n, qr, n, lane);
        if (t == 0) {
            out_id[q] = (int64_t)lo_id;
            out_dist[q] = __double2float_rn(sqrt(d));
        }
        return;
    }
    // pass 3: exact keys of the eligible rows, lexicographic minimum of (exact d^2, id)
    uint32_t best[XK], cur[XK];
    uint32_t best_id = 0xffffffffu;
    double best_d = INF64;
#pragma unroll
    for (int i = 0; i < XK; i++) best[i] = 0xffffffffu;
    for (uint32_t k = warp; k < cnt; k += NWF) {
        const NearEntry e = list[k];
        const double d = d64_of(k, e);
        if (!(d <= elig)) continue;
        exact_key(stored + (uint64_t)e.pos * n, qr, n, lane, cur);
        if (key_id_less(cur, e.id, best, best_id)) {
#pragma unroll
            for (int i = 0; i < XK; i++) best[i] = cur[i];
            best_id = e.id;
            best_d = d;
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < XK; i++) s_key[warp][i] = best[i];
        s_id[warp] = best_id;
        s_d64[warp] = best_d;
    }
    __syncthreads();
    if (t == 0) {
        uint32_t bw = 0;
        for (uint32_t w = 1; w < NWF; w++) {
            bool less = false, decided = false;
            for (int i = XK - 1; i >= 0 && !decided; i--)
                if (s_key[w][i] != s_key[bw][i]) {
                    less = s_key[w][i] < s_key[bw][i];
                    decided = true;
                }
            if (!decided) less = s_id[w] < s_id[bw];
            if (less) bw = w;
        }
        out_id[q] = (int64_t)s_id[bw];
        out_dist[q] = __double2float_rn(sqrt(s_d64[bw]));
    }
}

void launch_finalize(const isax_index *ix, uint32_t nq, const uint32_t *qmap, float delta, int64_t *out_id,
                     float *out_dist, cudaStream_t s) {
    const QueryScratch &qs = ix->qs;
    if (!nq) return;
    finalize_kernel<<<nq, FZ_THREADS, 0, s>>>(ix->stored, ix->n, qs.qy, qmap, qs.bsf,
                                              NearList{qs.near, qs.near_off, qs.near_cap, qs.near_cnt}, 1.0f + delta,
                                              out_id, out_dist);
}

}  // namespace isax
