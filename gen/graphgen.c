/*
 * gen/graphgen.c -- seeded synthetic graph generators (INPUT GENERATION ONLY).
 *
 * This module holds none of QQA's arithmetic. It produces the graph instances
 * that stand in for the paper's workloads (§5.1 "Erdős–Rényi graphs",
 * "regular random graphs (RRGs) with d = 100 and d = 20", Appendix E Table 12)
 * and is shared, read-only, by the CUDA path's tests/bench and by the oracle.
 *
 * RNG: SplitMix64 stream (state += golden gamma; output = mix(state)).
 *
 *   gen_er_edges   : G(n, p) -- every unordered pair {i<j} kept independently
 *                    with probability p (geometric skipping over the pair list).
 *   gen_rrg_edges  : simple d-regular graph -- configuration model (random
 *                    stub matching) followed by degree-preserving double-edge
 *                    swaps that remove self-loops and multi-edges.  A full
 *                    restart essentially never succeeds at d=20.
 *   edges_to_csr   : symmetric CSR, rows sorted ascending, no duplicates.
 *
 * Edges are returned as (u, v) pairs with u < v, each undirected edge once.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef struct { uint64_t s; } sm64;

static uint64_t sm64_next(sm64* r) {
    uint64_t z = (r->s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
/* uniform double in [0, 1) with 53 random bits */
static double sm64_unif(sm64* r) { return (double)(sm64_next(r) >> 11) * 0x1.0p-53; }
/* uniform integer in [0, n) (Lemire-free simple rejection; n > 0) */
static uint64_t sm64_below(sm64* r, uint64_t n) {
    uint64_t lim = UINT64_MAX - (UINT64_MAX % n);
    uint64_t x;
    do { x = sm64_next(r); } while (x >= lim);
    return x % n;
}

/* Public: one SplitMix64 output for a given counter (used for instance sizes). */
uint64_t gen_splitmix64(uint64_t x) {
    sm64 r = { x };
    return sm64_next(&r);
}

/* ---------------------------------------------------------------- ER ---- */
/* Returns number of edges written, or -(needed lower bound) if cap exceeded. */
int64_t gen_er_edges(int32_t n, double p, uint64_t seed, int32_t* eu, int32_t* ev, int64_t cap) {
    if (n < 2 || p <= 0.0) return 0;
    sm64 r = { seed };
    int64_t m = 0;
    if (p >= 1.0) {
        for (int32_t i = 0; i < n; ++i)
            for (int32_t j = i + 1; j < n; ++j) {
                if (m >= cap) return -(m + 1);
                eu[m] = i; ev[m] = j; ++m;
            }
        return m;
    }
    /* Walk the lexicographic pair list (i, j>i) with geometric skips. */
    const double lq = log1p(-p);
    int64_t i = 0, j = 0; /* current pair is (i, j); start before (0,1) */
    j = 0;
    for (;;) {
        double u = sm64_unif(&r);
        int64_t skip = (int64_t)floor(log1p(-u) / lq); /* failures before success */
        j += skip + 1;
        while (i < n && j >= n) { j = j - n + (i + 2); ++i; }
        if (i >= n - 1) break;
        if (m >= cap) return -(m + 1);
        eu[m] = (int32_t)i; ev[m] = (int32_t)j; ++m;
    }
    return m;
}

/* --------------------------------------------------------------- RRG ---- */
/* Adjacency as fixed d slots per node; a self-loop (a,a) fills two slots of a. */
static int has_edge(const int32_t* adj, int32_t d, int32_t a, int32_t b) {
    const int32_t* s = adj + (int64_t)a * d;
    for (int32_t k = 0; k < d; ++k) if (s[k] == b) return 1;
    return 0;
}
static int count_edge(const int32_t* adj, int32_t d, int32_t a, int32_t b) {
    const int32_t* s = adj + (int64_t)a * d;
    int c = 0;
    for (int32_t k = 0; k < d; ++k) c += (s[k] == b);
    return c;
}
static void replace_slot(int32_t* adj, int32_t d, int32_t a, int32_t oldb, int32_t newb) {
    int32_t* s = adj + (int64_t)a * d;
    for (int32_t k = 0; k < d; ++k) if (s[k] == oldb) { s[k] = newb; return; }
}
/* edge e is "bad" if it is a loop or has a parallel copy */
static int edge_bad(const int32_t* adj, int32_t d, int32_t a, int32_t b) {
    if (a == b) return 1;
    return count_edge(adj, d, a, b) > 1;
}

/* Writes m = n*d/2 edges (u<v). Returns m, or -1 (bad args), -2 (repair failed). */
int64_t gen_rrg_edges(int32_t n, int32_t d, uint64_t seed, int32_t* eu, int32_t* ev) {
    if (n <= 0 || d < 0 || d >= n || ((int64_t)n * d) % 2 != 0) return -1;
    const int64_t m = (int64_t)n * d / 2;
    if (m == 0) return 0;
    sm64 r = { seed };
    int64_t ns = (int64_t)n * d;
    int32_t* stubs = (int32_t*)malloc(sizeof(int32_t) * ns);
    int32_t* adj = (int32_t*)malloc(sizeof(int32_t) * ns);
    int32_t* fill = (int32_t*)calloc(n, sizeof(int32_t));
    if (!stubs || !adj || !fill) { free(stubs); free(adj); free(fill); return -1; }
    for (int64_t k = 0; k < ns; ++k) stubs[k] = (int32_t)(k / d);
    for (int64_t k = ns - 1; k > 0; --k) { /* Fisher-Yates */
        int64_t t = (int64_t)sm64_below(&r, (uint64_t)(k + 1));
        int32_t x = stubs[k]; stubs[k] = stubs[t]; stubs[t] = x;
    }
    for (int64_t e = 0; e < m; ++e) {
        int32_t a = stubs[2 * e], b = stubs[2 * e + 1];
        eu[e] = a; ev[e] = b;
        adj[(int64_t)a * d + fill[a]++] = b;
        adj[(int64_t)b * d + fill[b]++] = a;
    }
    free(stubs); free(fill);
    /* Degree-preserving double-edge swaps until no loop / multi-edge remains. */
    int64_t budget = 1000 * (m + 100);
    for (int pass = 0; pass < 1000; ++pass) {
        int64_t nbad = 0;
        for (int64_t e = 0; e < m; ++e) {
            int32_t a = eu[e], b = ev[e];
            if (!edge_bad(adj, d, a, b)) continue;
            ++nbad;
            /* swap (a,b),(c,e2) -> (a,c),(b,e2') with a random partner edge */
            for (int tries = 0; tries < 1000 && budget > 0; ++tries, --budget) {
                int64_t f = (int64_t)sm64_below(&r, (uint64_t)m);
                if (f == e) continue;
                int32_t c = eu[f], g = ev[f];
                if (sm64_next(&r) & 1) { int32_t t2 = c; c = g; g = t2; }
                /* new edges (a,c) and (b,g) must be simple and not yet present */
                if (a == c || b == g) continue;
                if (has_edge(adj, d, a, c) || has_edge(adj, d, b, g)) continue;
                /* also (a,c) vs (b,g) identical pair */
                if ((a == b && c == g) || (a == g && b == c)) continue;
                replace_slot(adj, d, a, b, c);
                replace_slot(adj, d, b, a, g);
                replace_slot(adj, d, c, g, a);
                replace_slot(adj, d, g, c, b);
                eu[e] = a; ev[e] = c;
                eu[f] = b; ev[f] = g;
                break;
            }
        }
        if (nbad == 0) break;
        if (budget <= 0) { free(adj); return -2; }
    }
    /* final verification */
    for (int64_t e = 0; e < m; ++e)
        if (edge_bad(adj, d, eu[e], ev[e])) { free(adj); return -2; }
    free(adj);
    for (int64_t e = 0; e < m; ++e)
        if (eu[e] > ev[e]) { int32_t t2 = eu[e]; eu[e] = ev[e]; ev[e] = t2; }
    return m;
}

/* -------------------------------------------------------------- CSR ---- */
static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}
/* rowptr[n+1], colidx[2m]. Returns 0, or -1 on loop/out-of-range, -2 on duplicate. */
int edges_to_csr(int32_t n, int64_t m, const int32_t* eu, const int32_t* ev,
                 int64_t* rowptr, int32_t* colidx) {
    memset(rowptr, 0, sizeof(int64_t) * ((size_t)n + 1));
    for (int64_t e = 0; e < m; ++e) {
        int32_t a = eu[e], b = ev[e];
        if (a < 0 || b < 0 || a >= n || b >= n || a == b) return -1;
        rowptr[a + 1]++; rowptr[b + 1]++;
    }
    for (int32_t i = 0; i < n; ++i) rowptr[i + 1] += rowptr[i];
    int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
    if (!pos) return -3;
    memcpy(pos, rowptr, sizeof(int64_t) * ((size_t)n + 1));
    for (int64_t e = 0; e < m; ++e) {
        colidx[pos[eu[e]]++] = ev[e];
        colidx[pos[ev[e]]++] = eu[e];
    }
    free(pos);
    for (int32_t i = 0; i < n; ++i) {
        int64_t a = rowptr[i], b = rowptr[i + 1];
        if (b - a > 1) qsort(colidx + a, (size_t)(b - a), sizeof(int32_t), cmp_i32);
        for (int64_t k = a + 1; k < b; ++k) if (colidx[k] == colidx[k - 1]) return -2;
    }
    return 0;
}
