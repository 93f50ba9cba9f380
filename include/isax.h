/* isax.h: C-ABI of libisax.so, exact 1-NN Euclidean search over iSAX-summarised data series
 * on one B200 (sm_100a).
 *
 * Method: ParIS / ParIS+ / MESSI, "Data Series Indexing Gone Parallel" (arXiv 2009.01614).
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; R<k> = the reading recorded in
 * DESIGN.md "Readings".
 *
 * Conventions (all entry points)
 *  - Series are row-major fp32 [count][n]. Sizes are element counts.
 *  - Pointers may be host (pageable or pinned) or device, unless a function says otherwise.
 *    The kind is detected with cudaPointerGetAttributes.
 *  - Inputs are borrowed for the duration of the call only. They are never modified or
 *    retained.
 *  - Return: ISAX_OK (0) or a negative ISAX_E_* code. On error, out-parameters are left
 *    untouched and isax_last_error() returns a thread-local message.
 *  - One index may be used by one host thread at a time; calls on the same index are
 *    serialised by an internal mutex. Separate indices are independent.
 *  - Environment: ISAX_DEBUG_ROUNDS=<k> prints the round plan's state (band, positions, counts) of every
 *    k-th round of a batch to stderr (diagnosis of slow overflow rounds; read once per process).
 *  - v1 supports w = 16, card = 256, n a multiple of 64 in [64, 1024], N < 2^32 - 1.
 *    Other valid arguments return ISAX_E_UNSUPPORTED.
 */
#ifndef ISAX_H
#define ISAX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    ISAX_OK = 0,
    ISAX_E_INVAL = -1,       /* bad argument: NULL pointer, n % w != 0, card not a power of 2 */
    ISAX_E_EMPTY = -2,       /* N == 0: an empty collection has no answer */
    ISAX_E_UNSUPPORTED = -3, /* valid by the method, outside what v1 implements */
    ISAX_E_NOMEM = -4,       /* a device or pinned allocation failed */
    ISAX_E_CUDA = -5,        /* a CUDA runtime error; the message names it */
    ISAX_E_NONFINITE = -6,   /* NaN or Inf in a series or a query */
    ISAX_E_CALLBACK = -7,    /* a fill callback returned non-zero */
    ISAX_E_IO = -8           /* isax_save / isax_load: the file cannot be opened, written or read in full */
};

/* Tunables. Pass NULL for the defaults. */
typedef struct isax_opts {
    uint32_t window_L;   /* rows of the approximate answer's main window (R5, R6b): whole
                            super-nodes around the query key's. Default 3072: it, the one before and the one after.
                            Range [1, 4096]; below 1024, a kd cell of the key's super-node. */
    int32_t slack_log2;  /* prune/abandon slack delta = 2^slack_log2 (R8). Default -12. */
    uint32_t batch_Q;    /* queries processed per device batch (<= 1024). Default 1024. */
    uint32_t cand_cap;   /* candidate-list capacity per query per round. 0 = default: a pool of 2^30 entries (about
                            12 B each; halved while it does not fit) split over the queries of each batch, at most
                            min(N, 2^23) per query. Overflow runs more rounds (R10): about 5 x candidates /
                            cand_cap of them, each a rescan, so a capacity far below a query's candidate
                            count is slow (5 over 220K series: about 120K rounds). */
    uint32_t flags;      /* ISAX_FLAG_* bits; 0 = defaults */
    uint32_t probe_bits; /* multi-probe approximate answer (R5): refine extra windows at the 2^probe_bits - 1 keys
                            obtained by flipping the most fragile plane-0/1 key bits; a probe window inside the main
                            window, or at the start of an earlier one, is skipped. 0 = default 5 (max);
                            ISAX_PROBES_NONE = main window only. */
    uint32_t probe_L;    /* rows per probe window: the kd cell of that many rows in the probe key's super-node
                            that the probe's symbols descend to (R6b). 0 = default 128, or 64 in a best-first
                            batch (first_band, R15). */
    float first_band;    /* best-first scan order (R15): round 0 scans only the smallest bounds,
                            LB^2 <= first_band * bsf0^2 (1 + delta), refines them, and the next round scans
                            the rest under the improved BSF; only the queries whose scan under the whole
                            threshold would keep more than 1/16 of the super-nodes get the fraction, the
                            others are scanned completely in round 0; with window_L = 0 the main window is
                            then a 512-row kd cell (and with probe_L = 0 each probe window 64 rows). 0 = adaptive
                            (default): fraction 1/50 or none, whichever the index measured to be faster per
                            query (device time); the other mode is re-timed after
                            32, 64, ... up to 512 batches while the choice holds. In (0, 1) = always, that
                            fraction; < 0 = never. Answers do not depend on it. */
} isax_opts;

#define ISAX_PROBES_NONE 0xFFFFFFFFu

/* opts.flags: scan every summary with no leaf pruning (the ParIS flat scan) instead
 * of the default leaf-pruned scan (MESSI's node pruning). The answers are identical;
 * this exists for A/B measurement. */
#define ISAX_FLAG_FLAT_SCAN 1u

typedef struct isax_index isax_index; /* opaque; owns all of its device memory */

/* Fill callback for isax_build_stream. It writes `count` raw series (ids first_id ..
 * first_id+count-1) into the DEVICE buffer dev_dst, [count][n] fp32, on cuda_stream (a
 * cudaStream_t). It must return 0 on success. It is called twice per chunk, in id order
 * (pass 1 summarises, pass 2 scatters), so it must produce the same bytes both times. */
typedef int (*isax_fill_fn)(void *ctx, uint64_t first_id, uint64_t count, float *dev_dst, void *cuda_stream);

/* Build an index over N raw series (north_star (a); P:289-336 MESSI stages 1-2, done as a
 * summarise + sort instead of a pointer tree).
 *  series : [N][n] fp32 raw values, host or device.
 *  w      : PAA segments; must divide n. v1: 16.
 *  card   : symbols per segment, a power of 2 in [2, 256]. v1: 256 (8 bits).
 *  opts   : NULL for defaults.
 *  out    : receives the index; free it with isax_free.
 * Each series is z-normalised (R2), summarised by PAA then SAX (R3, R4), and keyed by its
 * plane-interleaved iSAX word (R6). The z-normalised rows are stored on the device in ascending
 * (key, id) order, with every full block of 1024 positions (a super-node) reordered by a kd
 * split down to 32-row leaves (R6b): the SAX-sorted, leaf-contiguous layout.
 * Errors: E_EMPTY if N == 0; E_INVAL; E_UNSUPPORTED; E_NONFINITE; E_NOMEM; E_CUDA. */
int isax_build(const float *series, uint64_t N, uint32_t n, uint32_t w, uint32_t card,
               const isax_opts *opts, isax_index **out);

/* Same as isax_build, but the raw series come from `fill`, `chunk` series at a time (0 = a
 * default). This is for collections whose raw copy cannot sit next to the index in HBM:
 * BASELINE.json configs 3 and 4, 102.4 GB each. */
int isax_build_stream(uint64_t N, uint32_t n, uint32_t w, uint32_t card, isax_fill_fn fill, void *ctx,
                      uint64_t chunk, const isax_opts *opts, isax_index **out);

/* Exact 1-NN of Q raw queries (north_star (b)).
 *  queries  : [Q][n] fp32 raw; each is z-normalised by the build's rule.
 *  out_id   : [Q] int64, the original 0-based id of the nearest series. Ties go to the lowest id.
 *  out_dist : [Q] fp32, sqrt of the squared Euclidean distance between the z-normalised
 *             query and that series.
 * Any pointer kinds. Synchronous: it returns when the outputs are written. Q == 0 is a no-op.
 * The answers do not depend on Q, batching or stream. */
int isax_nn1(const isax_index *ix, const float *queries, uint32_t Q, int64_t *out_id, float *out_dist);

/* Same as isax_nn1 with DEVICE pointers, enqueued on cuda_stream (a cudaStream_t; NULL =
 * the legacy default stream). It synchronises the stream once per batch of opts.batch_Q
 * queries, to read the candidate-overflow flags. */
int isax_nn1_async(const isax_index *ix, const float *d_queries, uint32_t Q, int64_t *d_out_id,
                   float *d_out_dist, void *cuda_stream);

/* Copy index contents to caller buffers (any pointer kinds, NULL = skip):
 *  sax_by_id [count][w] u8: the iSAX words of ids first_id .. first_id+count-1.
 *  perm      [N] u32: perm[pos] = id of the series stored at sorted position pos.
 *  stored    [count][n] fp32: the z-normalised rows at sorted positions first_id .. +count-1.
 * Errors: E_INVAL if first_id + count > N. */
int isax_export(const isax_index *ix, uint64_t first_id, uint64_t count, uint8_t *sax_by_id, uint32_t *perm,
                float *stored);

/* Debug / parity entry: the query-side summaries and bounds the path uses.
 *  q_paa  [Q][w] fp64 (NULL = skip), q_sax [Q][w] u8 (NULL = skip),
 *  lut    [Q][w][card] fp32 (NULL = skip): (n/w) * mindist^2 per segment and symbol, rounded down,
 *  lb2    [Q][count] fp32 (NULL = skip): LB^2 of sorted positions first_pos .. +count-1
 *         (S:117-125), accumulated as the scan kernel does.
 *  win    [Q][2] u32 (NULL = skip): the approximate-answer window [start, end) (R5).
 * Any pointer kinds. */
int isax_query_debug(const isax_index *ix, const float *queries, uint32_t Q, double *q_paa, uint8_t *q_sax,
                     float *lut, uint64_t first_pos, uint64_t count, float *lb2, uint32_t *win);

/* Debug / parity entry: the candidate list of query q (0-based in the last isax_nn1 /
 * isax_nn1_async call) after the LB filter (the series "not pruned" by their lower
 * bound), as sorted positions, in no particular order. These are the positions p outside the
 * approximate answer's window with LB^2(p) <= bsf0^2 (1 + delta), bsf0 = the window's BSF
 * (R8, R10). *count receives the list length; out_pos (any pointer kind, or NULL to query the
 * length) receives it when cap >= *count.
 * Errors: E_INVAL if the last call spanned more than one batch (Q > batch_Q) or ran more than
 * one scan round (an overflowed list: the round's candidates are not kept). */
int isax_debug_candidates(const isax_index *ix, uint32_t q, uint32_t *out_pos, uint64_t cap, uint64_t *count);

/* Debug / test entry (host only, no device): one step of the per-query plan of scan rounds
 * (R9, R10; csrc/round_plan.h). In/out: band_lo_hi = the band (lo, hi] of LB^2, band_pos = its
 * sorted-position range [plo, phi), state = {length of the next position range, consecutive
 * first-bin overflows}. In: the round's candidate count and list capacity, its 64-bin histogram of
 * kept LB^2 over [max(lo, 0), tused], whether the near list overflowed, tused = the threshold the
 * round used, bsf_lim = bsf^2 (1 + delta) now, N. Returns 0 = no more rounds, 1 = scan the
 * updated band again, 2 = near-list overflow (grow the list, start over), -1 = overflow at a
 * single position. */
int isax_debug_plan_round(float *band_lo_hi, uint32_t *band_pos, uint32_t *state, uint32_t cand_cnt, uint32_t cap,
                          const uint32_t *hist, int near_ovf, float tused, float bsf_lim, uint32_t N);

/* Debug / test entry (device): returns 1 if this build has the device-side bounds checks
 * (libisax_bounds.so, -DISAX_BOUNDS), else 0. With fire != 0 it launches one kernel whose check
 * fails: the bounds build then returns ISAX_E_CUDA (the trap leaves the CUDA context unusable, so
 * call it with fire != 0 only in a process of its own); the product build returns 0. */
int isax_debug_bounds(int fire);

/* Persistence (not in the paper's in-memory path; the on-disk ParIS pipeline, is out of scope: this
 * only spares a rebuild). isax_save writes the index's geometry and every device array (stored rows, words,
 * permutation, kd splits and node summaries) to `path` (host file name), chunked through a pinned buffer;
 * isax_load reads such a file onto the current device and returns an index that holds byte for byte what the
 * saved one held, so it returns the same answers. opts as for isax_build (NULL = defaults; the file stores
 * none). Errors: ISAX_E_IO (open / short read or write), ISAX_E_INVAL (not an index file, sizes inconsistent),
 * ISAX_E_UNSUPPORTED (a file of another layout version), ISAX_E_NOMEM. The file is as large as the index
 * (about 4n + 29 bytes per series). */
int isax_save(const isax_index *ix, const char *path);
int isax_load(const char *path, const isax_opts *opts, isax_index **out);

/* Counters of the last isax_nn1 / isax_nn1_async call, as a JSON object written to buf.
 * It holds per-query window, window_rows (rows the approximate answer refined), candidates,
 * refined, abandoned, skipped, rounds, near, leaves_alive and the BSF before and after the scan,
 * plus per-stage device milliseconds of the first batch, the bytes and LUT lookups the first scan
 * launch counted (scan_bytes_first_launch, scan_lookups_first_launch: 16 per node or member bound
 * computed), the bytes its refine passes read, and build_ms: the device milliseconds of the
 * build's stages (summarise, sort, kd order + node summaries, permute; available right after
 * isax_build). Returns the length needed (excluding NUL); truncates if cap is too small. */
int isax_stats(const isax_index *ix, char *buf, size_t cap);

/* Index geometry: any out pointer may be NULL. device_bytes = bytes the index holds on the device. */
int isax_info(const isax_index *ix, uint64_t *N, uint32_t *n, uint32_t *w, uint32_t *card, uint64_t *device_bytes);

void isax_free(isax_index *ix);      /* NULL-safe */
const char *isax_last_error(void);   /* thread-local message of the last failing call on this thread */
const char *isax_version(void);      /* "isax-b200 <semver> sm_100a" */

#ifdef __cplusplus
}
#endif
#endif /* ISAX_H */
