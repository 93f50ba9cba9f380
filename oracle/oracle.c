/* oracle.c: plain C + OpenMP oracle of the iSAX exact 1-NN path. TEST INFRASTRUCTURE ONLY.
 *
 * This file computes the same definitions as oracle/ref.py (C1 z-norm, C2 PAA, C4 SAX,
 * C7 brute-force 1-NN), so the tests and the CPU baseline can run them at the benchmark
 * sizes. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
 * may link it. It shares no code with paper_2009_01614_b200/.
 *
 * Build: gcc -std=c11 -O2 -fopenmp -ffp-contract=off -fno-fast-math -shared -fPIC.
 * -ffp-contract=off forbids fusing a*b+c into an FMA, and the absence of -ffast-math
 * forbids reassociation. So each fp64 sum below runs strictly left to right over the
 * points of one series (reading R3), exactly as written.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

/* C1: z-normalise one row. Returns 0, or -1 if the row holds NaN/Inf. */
static int znorm_row(const float *x, int n, float *y, double *mu_out, double *sd_out)
{
    double s = 0.0;
    for (int i = 0; i < n; i++) {
        if (!isfinite(x[i])) return -1;
        s += (double)x[i];
    }
    double mu = s / (double)n;
    double s2 = 0.0;
    for (int i = 0; i < n; i++) {
        double t = (double)x[i] - mu;
        s2 += t * t;
    }
    double sd = sqrt(s2 / (double)n);
    if (sd < 1e-12) {
        for (int i = 0; i < n; i++) y[i] = 0.0f;
    } else {
        for (int i = 0; i < n; i++) y[i] = (float)(((double)x[i] - mu) / sd);
    }
    if (mu_out) *mu_out = mu;
    if (sd_out) *sd_out = sd;
    return 0;
}

/* C2 + C4: segment means and symbols: #{k : beta_k <= m}. */
static void paa_sax_row(const float *y, int n, int w, const double *beta, int card,
                        double *m_out, uint8_t *sym_out)
{
    int seg = n / w;
    for (int s = 0; s < w; s++) {
        double acc = 0.0;
        for (int j = 0; j < seg; j++) acc += (double)y[s * seg + j];
        double m = acc / (double)seg;
        int c = 0;
        for (int k = 0; k < card - 1; k++) c += (beta[k] <= m);
        if (m_out) m_out[s] = m;
        sym_out[s] = (uint8_t)c;
    }
}

/* Summarise N rows of raw series: y (nullable), mu, sigma, paa (nullable), symbols.
 * Returns the number of rows holding NaN/Inf; their outputs are unspecified. */
int64_t orc_summarise(const float *x, int64_t N, int n, int w, const double *beta, int card,
                      float *y_out, double *mu, double *sigma, double *paa, uint8_t *sym)
{
    int64_t bad = 0;
#pragma omp parallel reduction(+ : bad)
    {
        float *tmp = (float *)malloc(sizeof(float) * (size_t)n);
#pragma omp for schedule(static)
        for (int64_t r = 0; r < N; r++) {
            float *y = y_out ? y_out + r * (int64_t)n : tmp;
            if (znorm_row(x + r * (int64_t)n, n, y, mu ? mu + r : NULL, sigma ? sigma + r : NULL)) {
                bad++;
                continue;
            }
            paa_sax_row(y, n, w, beta, card, paa ? paa + r * (int64_t)w : NULL, sym + r * (int64_t)w);
        }
        free(tmp);
    }
    return bad;
}

/* C7: brute-force scan of one chunk of RAW rows (ids id0 .. id0+m-1) against Q z-normalised
 * queries. Each row is z-normalised by znorm_row, then d^2 = sum_i (q_i - y_i)^2 in fp64.
 *
 * Per query it keeps best_d2[q] (running minimum) and a "near" list of up to K (id, d2) entries
 * with d2 <= best * (1 + rel) + 1e-300. Those entries are resolved exactly by the caller
 * (oracle/clib.py) with rationals. If an entry does not fit, ovf_d2[q] records the smallest
 * d2 dropped that way: the list is complete iff ovf_d2[q] > best_d2[q] * (1 + rel) + 1e-300 at
 * the end (a dropped entry outside the final band cannot be the answer). State (best_d2,
 * near_cnt, near_id, near_d2, ovf_d2) is carried across chunks; initialise best_d2 and ovf_d2
 * to +inf and the counts to 0.
 *
 * The per-row loop is blocked over queries (qt is the transposed query matrix [n][Q]) so the
 * accumulators for different queries are independent. Each accumulator still sums its own
 * terms left to right.
 */
static void near_insert(int K, double rel, double *best, int *cnt, int64_t *ids, double *d2s,
                        double *ovf, int64_t id, double d)
{
    if (d < *best) {
        *best = d;
        int j = 0;
        for (int i = 0; i < *cnt; i++)
            if (d2s[i] <= d * (1.0 + rel) + 1e-300) { ids[j] = ids[i]; d2s[j] = d2s[i]; j++; }
        *cnt = j;
    }
    if (d <= *best * (1.0 + rel) + 1e-300) {
        if (*cnt < K) { ids[*cnt] = id; d2s[*cnt] = d; (*cnt)++; }
        else if (d < *ovf) *ovf = d;
    }
}

int64_t orc_nn1_scan(const float *xraw, int64_t m, int n, int64_t id0, const float *qt, int Q,
                     int K, double rel, double *best_d2, int *near_cnt, int64_t *near_id,
                     double *near_d2, double *ovf_d2)
{
    int64_t bad = 0;
#pragma omp parallel reduction(+ : bad)
    {
        float *y = (float *)malloc(sizeof(float) * (size_t)n);
        double *acc = (double *)malloc(sizeof(double) * (size_t)Q);
        double *lb = (double *)malloc(sizeof(double) * (size_t)Q);
        int *lc = (int *)calloc((size_t)Q, sizeof(int));
        int64_t *li = (int64_t *)malloc(sizeof(int64_t) * (size_t)Q * K);
        double *ld = (double *)malloc(sizeof(double) * (size_t)Q * K);
        double *lo = (double *)malloc(sizeof(double) * (size_t)Q);
        for (int q = 0; q < Q; q++) lb[q] = INFINITY, lo[q] = INFINITY;
#pragma omp for schedule(static)
        for (int64_t r = 0; r < m; r++) {
            if (znorm_row(xraw + r * (int64_t)n, n, y, NULL, NULL)) { bad++; continue; }
            for (int q = 0; q < Q; q++) acc[q] = 0.0;
            for (int i = 0; i < n; i++) {
                const float *qi = qt + (int64_t)i * Q;
                double yi = (double)y[i];
                for (int q = 0; q < Q; q++) {
                    double d = (double)qi[q] - yi;
                    acc[q] += d * d;
                }
            }
            for (int q = 0; q < Q; q++)
                near_insert(K, rel, &lb[q], &lc[q], li + (int64_t)q * K, ld + (int64_t)q * K, &lo[q],
                            id0 + r, acc[q]);
        }
#pragma omp critical
        {
            for (int q = 0; q < Q; q++) {
                if (lo[q] < ovf_d2[q]) ovf_d2[q] = lo[q];
                for (int i = 0; i < lc[q]; i++)
                    near_insert(K, rel, &best_d2[q], &near_cnt[q], near_id + (int64_t)q * K,
                                near_d2 + (int64_t)q * K, &ovf_d2[q], li[(int64_t)q * K + i],
                                ld[(int64_t)q * K + i]);
            }
        }
        free(y); free(acc); free(lb); free(lc); free(li); free(ld); free(lo);
    }
    return bad;
}

int orc_num_threads(void) { return omp_get_max_threads(); }
