/* examples/nn1_c.c: the C ABI from plain C (no Python, no torch).
 *
 * Builds an index over N random walks held in host memory, answers Q queries through the
 * synchronous isax_nn1 (host buffers), and checks every answer against a brute-force scan in
 * double precision written here. Prints one line per query and "ok" or "MISMATCH".
 *
 *   gcc -O2 -std=c99 -I include examples/nn1_c.c -L paper_2009_01614_b200 -lisax \
 *       -Wl,-rpath,$PWD/paper_2009_01614_b200 -lm -o /tmp/nn1_c && /tmp/nn1_c 20000 256 8
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "isax.h"

static uint64_t rng_state = 88172645463325252ull;
static double uniform01(void) { /* xorshift64*, (0, 1] */
    rng_state ^= rng_state >> 12;
    rng_state ^= rng_state << 25;
    rng_state ^= rng_state >> 27;
    return ((rng_state * 2685821657736338717ull) >> 11) * (1.0 / 9007199254740992.0) + 1e-300;
}
static double normal(void) { return sqrt(-2.0 * log(uniform01())) * cos(6.283185307179586 * uniform01()); }

static void walk(float *x, uint32_t n) {
    double v = 0.0;
    for (uint32_t i = 0; i < n; i++) x[i] = (float)(v += normal());
}

/* z-normalisation as the library defines it (R2): population sigma; sigma < 1e-12 -> zeros */
static void znorm(const float *x, double *y, uint32_t n) {
    double mu = 0.0, s2 = 0.0;
    for (uint32_t i = 0; i < n; i++) mu += x[i];
    mu /= n;
    for (uint32_t i = 0; i < n; i++) s2 += (x[i] - mu) * (x[i] - mu);
    const double sd = sqrt(s2 / n);
    for (uint32_t i = 0; i < n; i++) y[i] = sd < 1e-12 ? 0.0 : (double)(float)((x[i] - mu) / sd);
}

int main(int argc, char **argv) {
    const uint64_t N = argc > 1 ? strtoull(argv[1], 0, 10) : 20000;
    const uint32_t n = argc > 2 ? (uint32_t)atoi(argv[2]) : 256;
    const uint32_t Q = argc > 3 ? (uint32_t)atoi(argv[3]) : 8;
    float *x = malloc(sizeof(float) * N * n), *q = malloc(sizeof(float) * Q * n);
    for (uint64_t i = 0; i < N; i++) walk(x + i * n, n);
    for (uint32_t j = 0; j < Q; j++) walk(q + (uint64_t)j * n, n);
    isax_index *ix = NULL;
    if (isax_build(x, N, n, 16, 256, NULL, &ix) != ISAX_OK) {
        fprintf(stderr, "isax_build: %s\n", isax_last_error());
        return 2;
    }
    int64_t *id = malloc(sizeof(int64_t) * Q);
    float *dist = malloc(sizeof(float) * Q);
    if (isax_nn1(ix, q, Q, id, dist) != ISAX_OK) {
        fprintf(stderr, "isax_nn1: %s\n", isax_last_error());
        return 2;
    }
    double *y = malloc(sizeof(double) * n), *qy = malloc(sizeof(double) * n);
    int bad = 0;
    for (uint32_t j = 0; j < Q; j++) {
        znorm(q + (uint64_t)j * n, qy, n);
        double best = INFINITY;
        int64_t arg = -1;
        for (uint64_t i = 0; i < N; i++) {
            znorm(x + i * n, y, n);
            double d2 = 0.0;
            for (uint32_t k = 0; k < n && d2 <= best; k++) d2 += (y[k] - qy[k]) * (y[k] - qy[k]);
            if (d2 < best) {  /* strict: ties keep the lowest id */
                best = d2;
                arg = (int64_t)i;
            }
        }
        const int ok = arg == id[j] && fabs(sqrt(best) - dist[j]) <= 1e-5 * fmax(sqrt(best), 1e-3);
        printf("query %u: id %lld dist %.6f  (brute force %lld %.6f) %s\n", j, (long long)id[j], dist[j], (long long)arg,
               sqrt(best), ok ? "ok" : "MISMATCH");
        bad += !ok;
    }
    isax_free(ix);
    printf("%s\n", bad ? "MISMATCH" : "ok");
    return bad ? 1 : 0;
}
