// isax_internal.cuh: shared declarations of the libisax.so translation units (not part of the ABI).
//
// Data layout in HBM, per index:
//   stored [N][n] fp32  z-normalised rows, in ascending (key, id) order (sorted position = pos)
//   sax    [N][16] u8   iSAX word of the row at pos (16 B per series, one uint4 load)
//   perm   [N] u32      perm[pos] = original id
// The 16 breakpoints' worth of state a query needs (LUT) is built per query batch.
#pragma once
#include <cstdint>
#include <cstddef>
#include <mutex>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/isax.h"

// Device-side bounds checks, compiled in only with -DISAX_BOUNDS (libisax_bounds.so, built next to
// the product library and run by tests/test_bounds.py over the GPU parity suite): a failed check
// prints the condition and traps, so the call returns ISAX_E_CUDA instead of touching memory
// outside its arrays. The product build compiles them to nothing.
#ifdef ISAX_BOUNDS
#define ISAX_BOUND(cond)                                                                      \
    do {                                                                                      \
        if (!(cond)) {                                                                        \
            printf("isax bounds check failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);     \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define ISAX_BOUND(cond) \
    do {                 \
    } while (0)
#endif

namespace isax {

constexpr int W = 16;        // segments ("w is fixed to 16")
constexpr int CARD = 256;    // symbols per segment (8 bits)
constexpr int NEAR_K = 256;  // near-tie list capacity per query, until it overflows (R9; api.cu grows it)
constexpr uint32_t MAX_PROBES = 32;  // 2^probe_bits windows per query, probe_bits <= 5
constexpr uint32_t HIST_BINS = 64;   // per-query histogram of kept LB^2 inside its band (R10)
constexpr uint32_t LEAF_SIZE = 32;    // sorted positions per leaf node (R11)
constexpr uint32_t KD_CELL = 8;       // sorted positions per sub-leaf box: the kd cells of a leaf (R6b, R11c)
constexpr uint32_t SUPER_SIZE = 1024; // sorted positions per super-node (R11)
constexpr uint32_t HYPER_SIZE = 32768; // sorted positions per hyper-node (R11)
constexpr uint32_t B_UNCHECKED = 255;  // candq marker: the exact fp32 rule is still to be applied

// Packed BSF: high 32 bits = fp32 bits of d^2 (non-negative, so the bit order is the
// numeric order), low 32 bits = original id. atomicMin on the packed word is the
// lexicographic min of (d^2, id) (ties to the lowest id per north_star).
__host__ __device__ inline unsigned long long pack_bsf(float d2, uint32_t id) {
#ifdef __CUDA_ARCH__
    return ((unsigned long long)__float_as_uint(d2) << 32) | id;
#else
    uint32_t b;
    memcpy(&b, &d2, 4);
    return ((unsigned long long)b << 32) | id;
#endif
}

// The first four kd levels of a full super-node (R6b), heap order: node k (0..14) splits on
// segment s[k] & 0xFF, and its right half starts at the smallest symbol s[k] >> 8 of that segment
// there. s[15] == KD_NONE marks a super-node without kd splits (the partial last one).
constexpr uint16_t KD_NONE = 0xFFFFu;
constexpr uint32_t KD_LEVELS = 4;
struct __align__(16) KdSplits {
    uint16_t s[16];
};

struct NearEntry {  // a completed refinement within (1+delta) of the BSF at that moment (R9)
    uint32_t id;
    uint32_t pos;
    float d2;
    uint32_t pad;
};

// Query q's near list is near[near_off[q] .. near_off[q] + near_cap[q]). A batch starts with
// near_off[q] = q * NEAR_K and near_cap[q] = NEAR_K; a query whose list overflowed is given a
// region as large as twice the count it reached before its rescan (api.cu, R9).
struct NearList {
    NearEntry *base;
    const unsigned long long *off;
    const uint32_t *cap;
    uint32_t *cnt;
};

// One scan round of a query (R10): keep a position iff lo < LB^2 <= min(hi, bsf^2 (1 + delta))
// and plo <= pos < phi. The position range is [0, N) unless the LB band could not be split any
// further (many equal bounds): then the round covers part of the sorted positions.
struct __align__(16) Band {
    float lo, hi;
    uint32_t plo, phi;
};

// The per-batch status the host reads after every round: one contiguous block on the device and
// the same layout in pinned host memory, so a round ends with a single D2H copy.
struct StatusBlock {
    static constexpr size_t RESET_BYTES = 48;  // scan_bytes_dev, refine_bytes, flag (16-B slots)
    unsigned long long *bsf, *bsf_scan, *scan_bytes_dev, *refine_bytes;
    uint32_t *cand_cnt, *cand_cnt2, *cnt_hi, *near_cnt, *flag, *counters, *win, *leaves;
    // a multiple of 16: the host mirror's own arrays follow it (Band needs 16-byte alignment)
    static size_t bytes(uint32_t Q) { return ((size_t)Q * (8 + 8 + 4 * 4 + 16 + 8 + 4) + 16 * 16 + 15) & ~size_t(15); }
    void carve(void *base, uint32_t Q) {
        unsigned char *p = static_cast<unsigned char *>(base);
        auto take = [&](size_t n) { unsigned char *r = p; p += (n + 15) & ~size_t(15); return r; };
        bsf = reinterpret_cast<unsigned long long *>(take(8ull * Q));
        bsf_scan = reinterpret_cast<unsigned long long *>(take(8ull * Q));
        scan_bytes_dev = reinterpret_cast<unsigned long long *>(take(8));  // these three are zeroed
        refine_bytes = reinterpret_cast<unsigned long long *>(take(16));   // together: RESET_BYTES (2 passes)
        flag = reinterpret_cast<uint32_t *>(take(4));
        cand_cnt = reinterpret_cast<uint32_t *>(take(4ull * Q));
        cand_cnt2 = reinterpret_cast<uint32_t *>(take(4ull * Q));
        cnt_hi = reinterpret_cast<uint32_t *>(take(4ull * Q));
        near_cnt = reinterpret_cast<uint32_t *>(take(4ull * Q));
        counters = reinterpret_cast<uint32_t *>(take(16ull * Q));
        win = reinterpret_cast<uint32_t *>(take(8ull * Q));
        leaves = reinterpret_cast<uint32_t *>(take(4ull * Q));
    }
};

// Pinned host memory: the status mirror plus the per-round inputs the host writes.
struct HostMirror : StatusBlock {
    void *status = nullptr;
    uint32_t *qmap, *rewin, *hist, *near_cap;
    unsigned long long *near_off;
    Band *band;
    static size_t bytes(uint32_t Q) {
        return StatusBlock::bytes(Q) + (size_t)Q * (4 + 4 + 16 + 4 * HIST_BINS + 4 + 8) + 6 * 16;
    }
    void carve(void *base, uint32_t Q) {
        status = base;
        StatusBlock::carve(base, Q);
        unsigned char *p = static_cast<unsigned char *>(base) + StatusBlock::bytes(Q);
        auto take = [&](size_t n) { unsigned char *r = p; p += (n + 15) & ~size_t(15); return r; };
        band = reinterpret_cast<Band *>(take(16ull * Q));
        qmap = reinterpret_cast<uint32_t *>(take(4ull * Q));
        rewin = reinterpret_cast<uint32_t *>(take(4ull * Q));
        hist = reinterpret_cast<uint32_t *>(take(4ull * Q * HIST_BINS));
        near_cap = reinterpret_cast<uint32_t *>(take(4ull * Q));
        near_off = reinterpret_cast<unsigned long long *>(take(8ull * Q));
    }
};

// Per-batch scratch owned by the index (sized for opts.batch_Q queries).
struct QueryScratch {
    uint32_t cap_Q = 0;
    uint32_t cand_cap_slot = 0;  // allocated list entries per query slot (cap_Q slots)
    uint32_t cand_cap = 0;       // the current batch's capacity per query (<= cand_cap_slot * cap_Q / B)
    float *qy = nullptr;            // [Q][n] z-normalised queries
    double *qpaa = nullptr;         // [Q][16]
    uint8_t *qsax = nullptr;        // [Q][16]
    float *lut = nullptr;           // [Q][16][256] fp32, rounded down
    uint8_t *lut8 = nullptr;        // [Q][16][256] u8 scan table of each active slot (R11b)
    uint8_t *lut8c = nullptr;       // [Q][8][256] u8 coarse table of each active slot: segment pairs at 4 bits (R17)
    uint4 *qconst = nullptr;        // [Q][2] scan constants of each active slot (band lo, T, window, positions)
    uint32_t *win = nullptr;        // [Q][2] window [start, end)
    uint32_t *pwin = nullptr;       // [Q][MAX_PROBES]: kept probe window starts (probe_L rows each), count last
    unsigned long long *bsf = nullptr;  // [Q] packed
    uint32_t *cand = nullptr;       // [Q][cand_cap] sorted positions
    uint16_t *candq = nullptr;      // [Q][cand_cap] u8 bounds of each candidate, b | (b2 << 8): b / qscale <= LB^2
                                    // (or B_UNCHECKED: kept on its u8 sum alone, exact rule pending), b2 / qscale <=
                                    // LB^2 of segments 8..15 (R16)
    uint32_t *cand2 = nullptr;      // [Q][cand_cap] the candidates after candcheck_kernel (the refine's list)
    uint16_t *candq2 = nullptr;     // [Q][cand_cap] their bounds (as candq)
    uint32_t *cand_cnt2 = nullptr;  // [Q] first refine pass: cand2[q][0 .. cand_cnt2)
    uint32_t *cnt_hi = nullptr;     // [Q] second pass before filtering: cand2[q][cap - cnt_hi .. cap)
    uint32_t *cnt_f = nullptr;      // [Q] second pass after filtering: cand[q][0 .. cnt_f)
    float *qscale = nullptr;        // [Q] 254 / T of the query's last scan, rounded down (R11b)
    float *qT = nullptr;            // [Q] T of the query's last scan
    uint32_t *cand_cnt = nullptr;   // [Q] (may exceed cand_cap: overflow)
    NearEntry *near = nullptr;      // near pool: [Q][NEAR_K], then the grown lists of overflowed queries
    uint64_t near_pool = 0;         // entries allocated in `near`
    uint64_t near_used = 0;         // entries handed out in the current batch
    unsigned long long *near_off = nullptr;  // [Q] first entry of query q's near list in the pool
    uint32_t *near_cap = nullptr;   // [Q] its capacity
    uint32_t *near_cnt = nullptr;   // [Q] appends so far (may exceed near_cap: overflow)
    uint32_t *qmap = nullptr;       // [Q] active slot -> batch slot, for re-scan rounds
    Band *qband = nullptr;          // [Q] LB band (lo, hi] and position range of each active slot (R10)
    uint32_t *cand_hist = nullptr;  // [Q][HIST_BINS] histogram of kept LB^2 in the band
    uint32_t *counters = nullptr;   // [Q][4]: refined, abandoned, skipped by the u8 bound, (unused)
    uint32_t *counters_leaf = nullptr;  // [Q]: (leaf, query) pairs that survived the node bound
    unsigned long long *scan_bytes_dev = nullptr;  // leaf words and leaf summaries the leaf scan read, bytes (all launches of a call)
    uint32_t *task_ctr = nullptr;              // work counter of the persistent leaf scan (v1 kernel)
    uint2 *scan_entries = nullptr;             // [scan_groups][ceil(N/SUPER_SIZE)] (super-node, query mask) kept by the node scan
    uint32_t *scan_ctl = nullptr;              // [scan_groups][4]: entries (heavy), claim cursor, work estimate, light entries of each query group
    uint32_t *qkept = nullptr;                 // [Q] super-nodes the node scan kept for each active slot (R15 per query)
    uint32_t scan_groups = 0;                  // groups allocated: ceil(cap_Q / 16) + 1
    unsigned long long *refine_bytes = nullptr;  // [2] bytes of rows the refine passes 1 and 2 read (all launches of a call)
    uint32_t *flag = nullptr;       // non-finite query flag
    void *status = nullptr;         // the device StatusBlock (bsf, bsf_scan, counters, ... point into it)
    unsigned long long *bsf_scan = nullptr;  // [Q] the BSF each query's last scan used (the window BSF in round 0)
    uint32_t *qmap2 = nullptr;      // [Q] slots whose window is re-refined
    void *h_mirror = nullptr;       // pinned host memory of hm
    HostMirror hm{};
};

struct StageTimes {
    float qprep = 0, window = 0, lbscan = 0, candcheck = 0, refine = 0, finalize = 0;
    float refine1 = 0, filter = 0, refine2 = 0;  // the refine's two passes and the filter between them (R14)
};

}  // namespace isax

struct isax_index {
    uint64_t N = 0;
    uint32_t n = 0, w = 0, card = 0;
    isax_opts opts{};
    int device = 0;
    float *stored = nullptr;
    uint8_t *sax = nullptr;
    uint32_t *perm = nullptr;
    uint4 *skey = nullptr;     // [ceil(N/SUPER_SIZE)] z key of each super-node's first z-order position (R6b)
    isax::KdSplits *ksplit = nullptr;  // [ceil(N/SUPER_SIZE)] first four kd levels of each full super-node (R6b)
    uint8_t *lmeta = nullptr;  // [ceil(N/LEAF_SIZE)][32]: per-leaf min (16 B) and max (16 B) symbols
    uint8_t *cmeta = nullptr;  // [ceil(N/LEAF_SIZE) * LEAF_SIZE / KD_CELL][32]: per-cell (sub-leaf box) min and max symbols (R11c)
    uint8_t *smeta = nullptr;  // [ceil(N/SUPER_SIZE)][32]: per-super-node min and max symbols
    uint8_t *hmeta = nullptr;  // [ceil(N/HYPER_SIZE)][32]: per-hyper-node min and max symbols
    size_t device_bytes = 0;
    isax::QueryScratch qs;
    std::mutex mu;
    // last-call statistics (host copies)
    std::vector<uint32_t> st_win, st_cand, st_refined, st_abandoned, st_skipped, st_winrows, st_rounds, st_near, st_leaves;
    std::vector<float> st_bsf0, st_bsf_final;
    isax::StageTimes st_ms;
    float st_build_ms[4] = {0, 0, 0, 0};  // device ms of the build's stages: summarise, sort, kd order + node summaries, permute
    uint64_t st_launches = 0;  // kernels launched by the last nn1 call
    uint32_t st_last_Q = 0;     // Q of the last nn1 call
    // R15 first-band policy (adaptive by default): the measured device ms per query of batches run
    // with and without the first band (-1 = not measured yet); the cheaper mode is used, the other
    // one re-measured after fb_every batches
    float fb_ms_on = -1.f, fb_ms_off = -1.f;
    uint32_t fb_n_on = 0, fb_n_off = 0;  // measurements taken of each mode
    bool win_auto = true;       // window_L left to the library (opts.window_L == 0)
    uint32_t win_L = 3072;      // main window rows of the current batch (R5; 1024 in best-first mode when auto)
    bool pr_auto = true;        // probe_L left to the library (opts.probe_L == 0)
    uint32_t pr_L = 128;        // probe window rows of the current batch (64 in best-first mode when auto)
    uint32_t fb_since = 0;       // batches since the other mode was last measured
    uint32_t fb_every = 32;      // re-time the other mode after this many batches (doubles while the choice holds)
    float st_fb_frac = 0.f;      // first-band fraction of the last call's first batch (0 = none)
    uint32_t st_fb_improved = 0; // its queries whose BSF the first band at least halved (stats)
    uint32_t st_fb_banded = 0;   // its queries that got the first band (R15 per query)
    uint64_t st_scan_bytes = 0, st_scan_bytes_first = 0;  // summary bytes the scan read (all / first launch)
    uint64_t st_refine_bytes_first = 0;                    // row bytes the first round's refine read (both passes)
    uint64_t st_refine1_bytes_first = 0, st_refine2_bytes_first = 0;  // ... per pass
    uint64_t st_scan_lookups_first = 0;                    // LUT lookups of the first scan launch, counted by the kernel (16 per node or member test)
    uint64_t st_leaf_pairs_first = 0, st_scan_q_first = 0; // (leaf, query) pairs kept / queries of the first scan
    cudaEvent_t ev[11] = {};
    // isax_nn1 (host pointers): one stream and device staging, grown on demand
    cudaStream_t io_stream = nullptr;
    float *io_q = nullptr;
    int64_t *io_id = nullptr;
    float *io_dist = nullptr;
    uint32_t io_cap = 0;
};

namespace isax {

// ---- error plumbing (api.cu) ----
int set_error(int code, const std::string &msg);
int cuda_error(cudaError_t e, const char *what);

#define ISAX_CUDA(call)                                            \
    do {                                                           \
        cudaError_t _e = (call);                                   \
        if (_e != cudaSuccess) return ::isax::cuda_error(_e, #call); \
    } while (0)

// ---- kernels' host launchers ----
// summarise.cu
// Pass 1 of the build over rows [0, count) of x (raw, device). Writes, for id = id0 + r:
// sax_by_id[id], key[id] (uint4, 128-bit interleaved), musig[id] (mu, sigma as double2),
// and sets *bad if a row holds NaN/Inf.
void launch_summarise(const float *x, uint64_t count, uint32_t n, uint64_t id0, uint8_t *sax_by_id,
                      uint4 *key, double2 *musig, uint32_t *bad, cudaStream_t s);
// sort.cu: stable LSD radix sort of (key, id) ascending. The input ids are iota. On return
// perm (= ids_out) holds ids in ascending (key, id) order. Scratch is allocated internally.
int radix_sort_keys(uint4 *keys, uint32_t *ids, uint64_t N, uint32_t *perm_out, cudaStream_t s);
// permute.cu
void launch_gather_rows(const float *x, const double2 *musig, const uint32_t *perm, uint64_t N, uint32_t n,
                        float *stored, cudaStream_t s);
void launch_scatter_rows(const float *x, uint64_t count, uint64_t id0, const double2 *musig, const uint32_t *inv,
                         uint32_t n, float *stored, cudaStream_t s);
void launch_gather_sax(const uint8_t *sax_by_id, const uint32_t *perm, uint64_t N, uint8_t *sax, cudaStream_t s);
void launch_invert_perm(const uint32_t *perm, uint64_t N, uint32_t *inv, cudaStream_t s);
void launch_export_sax(const uint8_t *sax, const uint32_t *inv, uint64_t first_id, uint64_t count, uint8_t *out,
                       cudaStream_t s);
// query.cu
// band0 > 0: round 0 scans only the first band LB^2 <= band0 * bsf0^2 (1 + delta) (R15)
void launch_qprep(const isax_index *ix, const float *queries, uint32_t Q, float band0, cudaStream_t s, uint32_t *bad);
uint32_t probe_bits(const isax_index *ix);
uint32_t window_probes(const isax_index *ix);  // probe-sized windows per query (incl. neighbour quarters)
void launch_window(const isax_index *ix, uint32_t Q, const uint32_t *qmap, float delta, cudaStream_t s);
void launch_lb_dump(const isax_index *ix, uint32_t Q, uint64_t first_pos, uint64_t count, float *out,
                    cudaStream_t s);
// lbscan.cu
void launch_leaf_meta(const uint8_t *sax, uint64_t N, uint8_t *cmeta, uint8_t *lmeta, uint8_t *smeta, uint8_t *hmeta, cudaStream_t s);
// permute.cu: the kd order inside every full super-node (R6b), the super-nodes' smallest keys and
// their first two kd splits (sax and perm are permuted in place)
void launch_superkd(uint8_t *sax, uint32_t *perm, uint64_t N, uint4 *skey, KdSplits *ksplit, cudaStream_t s);
// Scan all sorted positions for the nq queries qmap[0..nq), keeping band[i].lo < LB^2 <= min(band[i].hi,
// bsf^2 (1+delta)) and band[i].plo <= pos < band[i].phi for slot i. Returns the summary bytes it reads that the host can count (node
// summaries or flat words); the leaf scan adds its leaf-word and leaf-summary bytes to qs.scan_bytes_dev on the device.
uint64_t launch_lbscan(const isax_index *ix, uint32_t nq, uint32_t B, const uint32_t *qmap, const Band *band,
                       float delta, bool select_first_band, cudaStream_t s);
// lbscan.cu: the exact fp32 rule for the candidates the leaf scan kept on their u8 sum alone,
// and compaction of every list into cand2 / cand_cnt2 (the refine's input)
void launch_candcheck(const isax_index *ix, uint32_t Q, cudaStream_t s);
// refine.cu
// evs (NULL or 2 events): recorded after pass 1 and after the filter (stage timing)
void launch_refine(const isax_index *ix, uint32_t Q, float delta, cudaStream_t s, cudaEvent_t *evs);
// finalise the nq queries qmap[0 .. nq) (the ones the round scanned): exact near-tie resolution (R9)
void launch_finalize(const isax_index *ix, uint32_t nq, const uint32_t *qmap, float delta, int64_t *out_id, float *out_dist,
                     cudaStream_t s);

}  // namespace isax
