/* datagen/gen.c -- seeded, hash-defined synthetic inputs.
 *
 * This is the ONLY code shared by the oracle side and the CUDA side: it builds
 * the graphs, matrix values and dense X that both consume.  It holds none of the
 * method's arithmetic (no decomposition, no product).  Every random choice is a
 * splitmix64 hash of a counter, so any implementation regenerates bit-identical
 * inputs.
 *
 *   splitmix64(x): z = x + 0x9E3779B97F4A7C15; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9;
 *                  z = (z ^ (z >> 27)) * 0x94D049BB133111EB; return z ^ (z >> 31)
 *   RMAT(scale, ef, s): edge e, bit l: h = splitmix64(splitmix64(s) ^ (64 e + l)),
 *       r = (h >> 11) 2^-53; bit l of u = [r >= 0.76]; bit l of v = [0.57 <= r < 0.76 or r >= 0.95]
 *       (Graph500 a,b,c = 0.57, 0.19, 0.19).
 *   value(u,v) = (2048 + (splitmix64(s_val ^ (min<<32 | max)) >> 52)) / 4096   in [0.5, 1.5), dyadic
 *   X[i,j]     = (splitmix64(s_X ^ (i*k + j)) >> 48) / 65536                     in [0, 1), dyadic
 *
 * Build: gcc -O3 -fopenmp -shared -fPIC datagen/gen.c -o datagen/_lib/libdatagen.so
 */
#include <stdint.h>

static inline uint64_t sm64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

void dg_splitmix64(const uint64_t *in, uint64_t *out, int64_t n) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = sm64(in[i]);
}

/* scramble keys: key_v = splitmix64(splitmix64(s+1) ^ v); labels are ranks of (key, v). */
void dg_scramble_keys(int64_t n, uint64_t s, uint64_t *key) {
    const uint64_t base = sm64(s + 1);
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; ++v) key[v] = sm64(base ^ (uint64_t)v);
}

/* raw (unscrambled) R-MAT endpoints for edges [e0, e1). */
void dg_rmat_edges(int32_t scale, uint64_t s, int64_t e0, int64_t e1, int32_t *u, int32_t *v) {
    const uint64_t base = sm64(s);
#pragma omp parallel for schedule(static)
    for (int64_t e = e0; e < e1; ++e) {
        uint32_t uu = 0, vv = 0;
        for (int32_t l = 0; l < scale; ++l) {
            uint64_t h = sm64(base ^ ((uint64_t)e * 64u + (uint64_t)l));
            double r = (double)(h >> 11) * 0x1.0p-53;
            uint32_t bu = (r >= 0.76) ? 1u : 0u;
            uint32_t bv = ((r >= 0.57 && r < 0.76) || r >= 0.95) ? 1u : 0u;
            uu |= bu << l;
            vv |= bv << l;
        }
        u[e - e0] = (int32_t)uu;
        v[e - e0] = (int32_t)vv;
    }
}

/* symmetric dyadic values for entries (r[i], c[i]). */
void dg_values(const int32_t *r, const int32_t *c, int64_t nnz, uint64_t s_val, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nnz; ++i) {
        uint64_t a = (uint64_t)(uint32_t)r[i], b = (uint64_t)(uint32_t)c[i];
        uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
        uint64_t h = sm64(s_val ^ ((lo << 32) | hi));
        out[i] = (double)(2048u + (h >> 52)) / 4096.0;
    }
}

/* dense X rows [r0, r1) of an n x k matrix, row-major, as fp64 (exact in fp32 too). */
void dg_fill_x(int64_t r0, int64_t r1, int64_t k, uint64_t s_x, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = r0; i < r1; ++i)
        for (int64_t j = 0; j < k; ++j) {
            uint64_t h = sm64(s_x ^ ((uint64_t)i * (uint64_t)k + (uint64_t)j));
            out[(i - r0) * k + j] = (double)(h >> 48) / 65536.0;
        }
}

void dg_fill_x_f32(int64_t r0, int64_t r1, int64_t k, uint64_t s_x, float *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = r0; i < r1; ++i)
        for (int64_t j = 0; j < k; ++j) {
            uint64_t h = sm64(s_x ^ ((uint64_t)i * (uint64_t)k + (uint64_t)j));
            out[(i - r0) * k + j] = (float)((double)(h >> 48) / 65536.0);
        }
}

/* ---------------------------------------------------------------- canonical CSR
 * Drop self-loops, merge duplicate undirected edges, store both (a,b) and (b,a), rows and
 * columns sorted.  keys = (min << 32 | max) sorted by an LSD radix sort (16-bit digits),
 * deduplicated; a sequential scan in (lo, hi) order then fills every row in ascending column
 * order (entries c < r arrive from keys (c, r) before the keys (r, c') with c' > r). */
#include <stdlib.h>
#include <string.h>

static void radix_sort_u64(uint64_t *a, uint64_t *tmp, int64_t m, int bits) {
    int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * 65536);
    for (int shift = 0; shift < bits; shift += 16) {
        memset(cnt, 0, sizeof(int64_t) * 65536);
        for (int64_t i = 0; i < m; ++i) cnt[(a[i] >> shift) & 0xFFFF]++;
        int64_t s = 0;
        for (int d = 0; d < 65536; ++d) { int64_t c = cnt[d]; cnt[d] = s; s += c; }
        for (int64_t i = 0; i < m; ++i) tmp[cnt[(a[i] >> shift) & 0xFFFF]++] = a[i];
        uint64_t *t = a; a = tmp; tmp = t;
        memcpy(tmp, a, sizeof(uint64_t) * m);  /* keep result in both buffers */
    }
    free(cnt);
}

/* returns nnz (stored entries); row_ptr[n+1] filled; col must have room for 2*m entries */
int64_t dg_canonicalize(int64_t n, int64_t m, const int64_t *u, const int64_t *v, int64_t *row_ptr, int32_t *col) {
    uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (m > 0 ? m : 1));
    uint64_t *tmp = (uint64_t *)malloc(sizeof(uint64_t) * (m > 0 ? m : 1));
    int64_t k = 0;
    for (int64_t e = 0; e < m; ++e) {
        uint64_t a = (uint64_t)u[e], b = (uint64_t)v[e];
        if (a == b) continue;
        uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
        keys[k++] = (lo << 32) | hi;
    }
    int bits = 32;
    while (bits < 64 && (((uint64_t)n - 1) >> (bits - 32)) != 0) bits += 1;
    bits = ((bits + 15) / 16) * 16;
    radix_sort_u64(keys, tmp, k, bits);
    int64_t w = 0;
    for (int64_t i = 0; i < k; ++i)
        if (i == 0 || keys[i] != keys[i - 1]) keys[w++] = keys[i];
    for (int64_t r = 0; r <= n; ++r) row_ptr[r] = 0;
    for (int64_t i = 0; i < w; ++i) { row_ptr[(keys[i] >> 32) + 1]++; row_ptr[(keys[i] & 0xFFFFFFFFu) + 1]++; }
    for (int64_t r = 0; r < n; ++r) row_ptr[r + 1] += row_ptr[r];
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    for (int64_t r = 0; r < n; ++r) cur[r] = row_ptr[r];
    for (int64_t i = 0; i < w; ++i) {
        int64_t lo = (int64_t)(keys[i] >> 32), hi = (int64_t)(keys[i] & 0xFFFFFFFFu);
        col[cur[lo]++] = (int32_t)hi;
        col[cur[hi]++] = (int32_t)lo;
    }
    free(cur); free(keys); free(tmp);
    return row_ptr[n];
}
