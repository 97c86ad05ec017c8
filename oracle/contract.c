/*
 * oracle/contract.c -- QQA oracle, fp32 CONTRACT mode.   TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. The product path
 * (paper_2409_02135_b200/, libqqa.so) shares no code with it.
 *
 * Plain single-threaded loops (an optional OpenMP pragma over independent
 * rows does not change any arithmetic). Build: gcc -O2 -ffp-contract=off
 * (no FMA contraction, no fast-math); x86-64 SSE gives IEEE binary32/64.
 *
 * WHAT IT COMPUTES (PAPER.md lines "P:nnn"):
 *   p = sigmoid(theta)                                              P:143, BASELINE north_star
 *   dR/dp = dl/dp + gamma ds/dp + d(-S a_c sum STD)/dp               Eq. 6, 7, 10
 *     MIS / clique-as-MIS-on-complement: dl/dp_i = -1 + lam q_i
 *     Max-Cut:                          dl/dp_i = -deg_i + 2 q_i
 *     q_i = sum_{j in N(i)} p_j
 *     gamma ds/dp = -2 alpha gamma (2p - 1)^(alpha-1)
 *     comm: -a_c (p - mu_i) / STD_i  (0 if STD_i < 1e-6)              P:196-198, R6
 *   dR/dtheta = dR/dp * p (1 - p)
 *   AdamW, decoupled weight decay
 *   x = Theta(p - 1/2) evaluated as theta >= 0
 *   weighted graphs (A_ij = w_ij; MIS and Max-Cut): q_i = sum_j w_ij p_j summed as
 *     q = fl(q + fl(w_ij p_j)) in CSR order (w = 1 gives the unweighted sums bit for bit), the
 *     Max-Cut degree sum_j w_ij as ((0 + w_1) + w_2) + ...; evaluation sums of w as exact int64
 *     fixed point llrint(w 2^24)
 *   max clique, printed relaxation on the original graph (problem 4):
 *     dl/dp_i = -1 + lam ((T - 1/2) - q_i), T = sum_k p_k of the replica, as
 *     fl(fl(lam fl(fl(T_f - 1/2) - q)) - 1) with T_f = (float)((double)C 2^-40),
 *     C = sum_k llrint(p_k 2^40) (int64, exact)
 *   map = CLAMP (sensitive transition, NEXT-1): AdamW on p itself with
 *     dR/dp (no chain factor), then p = Clamp(p') into [0, 1]         Eq. 11
 *     x = Theta(p - 1/2) evaluated as p >= 1/2
 *   Langevin noise (NEXT-2): + sqrt(2 lr T) xi after the optimizer
 *     step, before the map; xi ~ N(0,1) by Box-Muller from a counter
 *     hash keyed (seed, t, i, s)                                     Eq. 9/11
 *   energies from integer counts
 *
 * THE fp32 CONTRACT: every element follows one fixed sequence
 * of IEEE round-to-nearest operations, so an implementation that performs the
 * same sequence gets bit-identical results:
 *   - gather q = ((0 + p_j1) + p_j2) + ...  in ascending CSR order;
 *   - sigmoid: exp by Cody-Waite reduction + degree-7 Taylor (Horner) in fp32
 *     (oc_exp_neg), p = 1/(1+E) for theta >= 0 else E/(1+E);
 *   - cross-replica stats as exact int64 fixed-point sums (scale 2^40) of
 *     d = p - c_i and fl(d*d), c_i = the previous step's mean (1/2 at init);
 *   - binary gradient: g_p = fma(p - mu_i, kc_i, fma(k_t, (2p-1)^(alpha-1), obj)) with the
 *     row's communication coefficient kc_i = fl(-a_c / STD_i) (0 if STD_i < 1e-6), one
 *     division per row (round 2; the K-ary rows keep -a_c ((p - mu) / STD) per element);
 *   - per-step scalars computed in double on the host, rounded to fp32.
 * The contract is pinned against the fp64 definition (oracle/definition.py)
 * in tests/test_oracle_contract.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OC_MIS = 0, OC_MAXCUT = 1, OC_MAXCLIQUE = 2, OC_MAXCLIQUE_SPARSE = 4 };

typedef struct {
    int32_t problem;     /* 0 MIS, 1 Max-Cut, 2 max clique (caller passes the complement CSR) */
    int32_t alpha;       /* entropy exponent (even >= 2) */
    float penalty;       /* lambda */
    float comm;          /* alpha_c, communication strength */
    float lr, beta1, beta2, eps, weight_decay;
    float init_lo, init_hi;
    uint64_t seed;
    int32_t S;           /* replicas (the oracle always holds all of them) */
    int32_t threads;     /* OpenMP threads for the row loop (<=1: serial) */
    int32_t map;         /* 0 sigmoid (theta is the parameter), 1 clamp (p is the parameter) */
    float temperature;   /* Langevin T; 0 = no noise */
    int32_t kary_grad;   /* K-ary: 1 = gradient through the map, g - <g, p> (reading R33); 0 = dR/dP (R29) */
} oc_cfg;

enum { OC_MAP_SIGMOID = 0, OC_MAP_CLAMP = 1 };

/* ------------------------------------------------------------ sigmoid ---- */
/* E = exp(-a) for 0 <= a <= 87, in fp32: a = k ln2 + r, exp(r) by Taylor. The reduction and the
 * Horner steps are fused multiply-adds (fmaf: one rounding, IEEE-exact on every platform, the GPU's
 * __fmaf_rn), the contract of DESIGN.md §3 item 2. */
float oc_exp_neg(float a) {
    const float x = -a;
    const float kf = rintf(x * 1.44269504088896341f);       /* nearest k */
    const float r = fmaf(-kf, 1.428606765330187e-6f,          /* ln2 lo */
                         fmaf(-kf, 0.693145751953125f, x));   /* ln2 hi */
    float P = 1.0f / 5040.0f;                                  /* 1/7! */
    P = fmaf(P, r, 1.0f / 720.0f);
    P = fmaf(P, r, 1.0f / 120.0f);
    P = fmaf(P, r, 1.0f / 24.0f);
    P = fmaf(P, r, 1.0f / 6.0f);
    P = fmaf(P, r, 1.0f / 2.0f);
    P = fmaf(P, r, 1.0f);
    P = fmaf(P, r, 1.0f);
    int k = (int)kf;                                           /* in [-126, 0] */
    union { uint32_t u; float f; } two_k;
    two_k.u = (uint32_t)(k + 127) << 23;
    return P * two_k.f;
}

float oc_sigmoid(float theta) {
    const float a = fabsf(theta);
    const float E = (a > 87.0f) ? 0.0f : oc_exp_neg(a);
    const float den = 1.0f + E;
    return (theta >= 0.0f) ? 1.0f / den : E / den;
}

void oc_sigmoid_array(int64_t n, const float* in, float* out) {
    for (int64_t k = 0; k < n; ++k) out[k] = oc_sigmoid(in[k]);
}

/* Clamp(w) into [0, 1]; NaN and -0 map to +0 (NaN is flagged before). */
float oc_clamp01(float w) {
    return (w > 0.0f) ? ((w < 1.0f) ? w : 1.0f) : 0.0f;
}

/* ------------------------------------------------------ Gaussian noise ---- */
/* ln(u), u in (0, 1], fp32: u = 2^e m, m in [sqrt(1/2), sqrt(2)), f = m - 1
 * (exact), s = f/(2+f), ln m = 2 atanh(s) = 2 s (1 + s^2/3 + s^4/5 + s^6/7 + s^8/9),
 * ln u = (e ln2_hi + ln m) + e ln2_lo. */
float oc_ln(float u) {
    union { float f; uint32_t u; } b;
    b.f = u;
    int e = (int)((b.u >> 23) & 0xffu) - 127;
    b.u = (b.u & 0x007fffffu) | 0x3f800000u;                   /* m in [1, 2) */
    float m = b.f;
    if (m > 1.41421356f) { m = m * 0.5f; e = e + 1; }
    const float f = m - 1.0f;
    const float s = f / (2.0f + f);
    const float z = s * s;
    float P = 1.0f / 9.0f;                                     /* Horner steps as fmaf (one rounding) */
    P = fmaf(P, z, 1.0f / 7.0f);
    P = fmaf(P, z, 1.0f / 5.0f);
    P = fmaf(P, z, 1.0f / 3.0f);
    P = fmaf(P, z, 1.0f);
    const float lnm = 2.0f * (s * P);
    const float ef = (float)e;
    return (ef * 0.693145751953125f + lnm) + ef * 1.428606765330187e-6f;
}

/* cos(2 pi x) and sin(2 pi x), x in [0, 1): y = 4x (exact), k = rint(y), r = y - k in
 * [-1/2, 1/2] (exact), a = r pi/2 in [-pi/4, pi/4]; from the Taylor polynomials of cos a (to a^8)
 * and sin a (to a^9) by quadrant k mod 4. */
void oc_cossin2pi(float x, float* c, float* sn) {
    const float y = 4.0f * x;
    const float k = rintf(y);
    const float r = y - k;
    const float a = r * 1.57079632679489662f;
    const float a2 = a * a;
    float C = 1.0f / 40320.0f;                                 /* Horner steps as fmaf (one rounding) */
    C = fmaf(C, a2, -(1.0f / 720.0f));
    C = fmaf(C, a2, 1.0f / 24.0f);
    C = fmaf(C, a2, -0.5f);
    C = fmaf(C, a2, 1.0f);
    float Sn = 1.0f / 362880.0f;
    Sn = fmaf(Sn, a2, -(1.0f / 5040.0f));
    Sn = fmaf(Sn, a2, 1.0f / 120.0f);
    Sn = fmaf(Sn, a2, -(1.0f / 6.0f));
    Sn = fmaf(Sn, a2, 1.0f);
    Sn = Sn * a;
    const int q = ((int)k) & 3;
    *c = (q == 0) ? C : (q == 1) ? -Sn : (q == 2) ? -C : Sn;
    *sn = (q == 0) ? Sn : (q == 1) ? C : (q == 2) ? -Sn : -C;
}

float oc_sin2pi(float x) {
    float c, sn;
    oc_cossin2pi(x, &c, &sn);
    return sn;
}

float oc_cos2pi(float x) {
    float c, sn;
    oc_cossin2pi(x, &c, &sn);
    return c;
}

/* Two independent N(0, 1) from one 64-bit hash h by Box-Muller:
 * u1 = (top 24 bits + 1) 2^-24 in (0, 1], u2 = (bits 16..39) 2^-24 in [0, 1),
 * r = sqrt(-2 ln u1); zc = r cos(2 pi u2), zs = r sin(2 pi u2). */
void oc_gauss_pair_from_hash(uint64_t h, float* zc, float* zs) {
    const float u1 = (float)((h >> 40) + 1u) * 0x1p-24f;
    const float u2 = (float)((h >> 16) & 0xFFFFFFu) * 0x1p-24f;
    const float r = sqrtf(-2.0f * oc_ln(u1));
    float c, sn;
    oc_cossin2pi(u2, &c, &sn);
    *zc = r * c;
    *zs = r * sn;
}

float oc_gauss_from_hash(uint64_t h) {
    float zc, zs;
    oc_gauss_pair_from_hash(h, &zc, &zs);
    return zc;
}

/* ------------------------------------------------------ step scalars ---- */
/* out = { k_t = -2 alpha gamma_t, a_t = 1 - lr wd, s_t = lr/(1-b1^t), r_t = 1/sqrt(1-b2^t) } */
void oc_step_scalars(const oc_cfg* c, int64_t t, float gamma_t, float* out) {
    out[0] = (float)(-2.0 * (double)c->alpha * (double)gamma_t);
    out[1] = (float)(1.0 - (double)c->lr * (double)c->weight_decay);
    out[2] = (float)((double)c->lr / (1.0 - pow((double)c->beta1, (double)t)));
    out[3] = (float)(1.0 / sqrt(1.0 - pow((double)c->beta2, (double)t)));
}

/* gamma_t = gmin + (gmax - gmin) t / (T - 1), t = 0..T-1 (reading R10) */
void oc_schedule(float gmin, float gmax, int64_t T, float* out) {
    for (int64_t t = 0; t < T; ++t)
        out[t] = (T == 1) ? gmin
                          : (float)((double)gmin + (((double)gmax - (double)gmin) * (double)t) / (double)(T - 1));
}

/* ----------------------------------------------------------- stats ------ */
static void finalize_stats(float c, int64_t sD, int64_t sD2, int32_t S, float* mu, float* sd) {
    const double md = ((double)sD * 0x1p-40) / (double)S;
    *mu = (float)((double)c + md);
    const double ex2 = ((double)sD2 * 0x1p-40) / (double)S;
    const double var = ex2 - md * md;
    *sd = (float)sqrt(var > 0.0 ? var : 0.0);
}

static void row_sums(const float* prow, int32_t S, float c, int64_t* sD, int64_t* sD2) {
    int64_t a = 0, b = 0;
    for (int32_t s = 0; s < S; ++s) {
        const float d = prow[s] - c;
        a += llrintf(d * 0x1p40f);
        const float dd = d * d;
        b += llrintf(dd * 0x1p40f);
    }
    *sD = a; *sD2 = b;
}

/* public: mean and STD of one row from its sums (for tests) */
void oc_finalize(float c, int64_t sD, int64_t sD2, int32_t S, float* mu_sd) {
    finalize_stats(c, sD, sD2, S, &mu_sd[0], &mu_sd[1]);
}

/* ------------------------------------------------------------ init ------ */
static uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Noise of (Adam step t, variable i, global replica s): replicas pair up (s even, s + 1) on
 * h = mix64(mix64(seed ^ 0x6A09E667F3BCC909) + (t n + i) S_total + s_even); xi = zc (s even) or
 * zs (s odd) of oc_gauss_pair_from_hash(h). */
uint64_t oc_noise_base(uint64_t seed) { return mix64(seed ^ 0x6A09E667F3BCC909ULL); }

float oc_noise(uint64_t base, int64_t t, int32_t n, int32_t i, int32_t S_total, int32_t s) {
    const uint64_t key = base + ((uint64_t)t * (uint64_t)n + (uint64_t)i) * (uint64_t)S_total + (uint64_t)(s & ~1);
    float zc, zs;
    oc_gauss_pair_from_hash(mix64(key), &zc, &zs);
    return (s & 1) ? zs : zc;
}

void oc_noise_array(uint64_t seed, int64_t t, int32_t n, int32_t S, float* out) {
    const uint64_t base = oc_noise_base(seed);
    for (int32_t i = 0; i < n; ++i)
        for (int32_t s = 0; s < S; ++s) out[(size_t)i * S + s] = oc_noise(base, t, n, i, S, s);
}

/* sqrt(2 lr T), the Langevin noise scale (Eq. 9, eta = lr), host double -> fp32 */
float oc_noise_scale(const oc_cfg* c) {
    return (float)sqrt(2.0 * (double)c->lr * (double)c->temperature);
}

/* theta_0 ~ U(lo, hi) by a counter hash keyed (seed, i, s); m = v = 0; p = sigmoid(theta);
 * c = 1/2; sums of p with shift 1/2. Arrays are [n][S] row-major.
 * map = CLAMP: the parameter is p itself, p_0 = 1/2 + U(lo, hi) (the same hash,
 * the sum formed in double and rounded once); theta holds p. */
void oc_init(int32_t n, const oc_cfg* cf, float* theta, float* m, float* v, float* p,
             float* c, int64_t* sumD, int64_t* sumD2) {
    const int32_t S = cf->S;
    const uint64_t base = mix64(cf->seed);
    const double lo = (double)cf->init_lo, hi = (double)cf->init_hi;
    for (int32_t i = 0; i < n; ++i) {
        for (int32_t s = 0; s < S; ++s) {
            const uint64_t key = base + (uint64_t)i * (uint64_t)S + (uint64_t)s;
            const uint64_t k = mix64(key) >> 40;
            const size_t at = (size_t)i * S + s;
            if (cf->map == OC_MAP_CLAMP) {
                theta[at] = (float)(0.5 + (lo + (hi - lo) * (double)k * 0x1p-24));
                p[at] = theta[at];
            } else {
                theta[at] = (float)(lo + (hi - lo) * (double)k * 0x1p-24);
                p[at] = oc_sigmoid(theta[at]);
            }
            m[at] = 0.0f;
            v[at] = 0.0f;
        }
        c[i] = 0.5f;
        row_sums(p + (size_t)i * S, S, 0.5f, &sumD[i], &sumD2[i]);
    }
}

/* ------------------------------------------------------------ one row --- */
/* Update row i. Reads p (old values, all rows) and the row's stats (c_i, sums);
 * updates th/mm/vv (row i, length S) in place; writes p_new (row i) and the
 * row's new stats (shift = this step's mean). */
static int update_row(int32_t i, int32_t n, int64_t t, const int64_t* rowptr, const int32_t* colidx,
                       const float* wts, const oc_cfg* cf, const float* sc, const float* Tcol, const float* p,
                       float* th, float* mm, float* vv,
                       float c_i, int64_t sD_i, int64_t sD2_i,
                       float* p_new, float* c_new, int64_t* sD_new, int64_t* sD2_new, float* q) {
    const int32_t S = cf->S;
    const float kt = sc[0], at = sc[1], st = sc[2], rt = sc[3];
    const float b1 = cf->beta1, b2 = cf->beta2, eps = cf->eps;
    const float c1 = (float)(1.0 - (double)cf->beta1), c2 = (float)(1.0 - (double)cf->beta2);
    const float lam = cf->penalty, ac = cf->comm;
    const int clamp = cf->map == OC_MAP_CLAMP;
    const float ns = oc_noise_scale(cf);
    const uint64_t nbase = oc_noise_base(cf->seed);
    const int64_t e0 = rowptr[i], e1 = rowptr[i + 1];
    float degf = (float)(e1 - e0);
    if (wts) {                                   /* weighted degree, CSR order */
        degf = 0.0f;
        for (int64_t e = e0; e < e1; ++e) degf = degf + wts[e];
    }
    const float* pown = p + (size_t)i * S;
    int nonfinite_flag = 0;

    float mu, sd;
    finalize_stats(c_i, sD_i, sD2_i, S, &mu, &sd);
    /* Eq. 10 gradient -alpha_c (p - mu) / STD as (p - mu) kc with the row's kc = -alpha_c / STD
     * (one division per row; 0 if STD < 1e-6, reading R6) */
    const float kc = (sd >= 1e-6f) ? (-ac) / sd : 0.0f;

    /* q_i^s = sum_{j in N(i)} p_j^s, ascending CSR order */
    for (int32_t s = 0; s < S; ++s) q[s] = 0.0f;
    for (int64_t e = e0; e < e1; ++e) {
        const float* pj = p + (size_t)colidx[e] * S;
        if (wts) {
            const float w = wts[e];
            for (int32_t s = 0; s < S; ++s) q[s] = q[s] + w * pj[s];
        } else {
            for (int32_t s = 0; s < S; ++s) q[s] = q[s] + pj[s];
        }
    }

    for (int32_t s = 0; s < S; ++s) {
        const float pi = pown[s];
        /* gradient dR/dp */
        const float e = 2.0f * pi - 1.0f;
        float ep = e;
        for (int32_t a = 2; a < cf->alpha; ++a) ep = ep * e;   /* (2p-1)^(alpha-1) */
        /* a * b + c written fmaf(a, b, c) is one fused multiply-add (one rounding) in the contract */
        const float obj = (cf->problem == OC_MAXCUT) ? fmaf(2.0f, q[s], -degf)
                          : (cf->problem == OC_MAXCLIQUE_SPARSE) ? fmaf(lam, (Tcol[s] - 0.5f) - q[s], -1.0f)
                          : fmaf(lam, q[s], -1.0f);
        const float gp = fmaf(pi - mu, kc, fmaf(kt, ep, obj));   /* (obj + entropy) + comm, fused */
        /* sigmoid: chain rule dR/dtheta = dR/dp p (1-p); clamp: the parameter is p */
        const float g = clamp ? gp : gp * (pi * (1.0f - pi));
        /* AdamW */
        float t1 = th[s] * at;
        const float m1 = fmaf(b1, mm[s], c1 * g);
        const float v1 = fmaf(b2, vv[s], (c2 * g) * g);
        const float den = fmaf(sqrtf(v1), rt, eps);
        t1 = fmaf(-st, m1 / den, t1);
        if (cf->temperature > 0.0f)                       /* Langevin noise, Eq. 9 / 11 */
            t1 = fmaf(ns, oc_noise(nbase, t, n, i, S, s), t1);
        if (!isfinite(t1)) nonfinite_flag = 1;            /* SPEC.md:396 abort, before the map */
        if (clamp) {
            t1 = oc_clamp01(t1);                          /* p^{t+1} = Clamp(p'), Eq. 11 */
            p_new[s] = t1;
        } else {
            p_new[s] = oc_sigmoid(t1);
        }
        th[s] = t1; mm[s] = m1; vv[s] = v1;
    }
    *c_new = mu;
    row_sums(p_new, S, mu, sD_new, sD2_new);
    return nonfinite_flag;
}

/* Per-replica column sums of p for the printed clique relaxation: T_s = (float)((double)C_s 2^-40),
 * C_s = sum_k llrint(p_ks 2^40) (exact int64, order-free). */
void oc_colsum(int32_t n, int32_t S, const float* p, float* T) {
    for (int32_t s = 0; s < S; ++s) {
        int64_t C = 0;
        for (int32_t k = 0; k < n; ++k) C += llrintf(p[(size_t)k * S + s] * 0x1p40f);
        T[s] = (float)((double)C * 0x1p-40);
    }
}

/* Run n_steps annealing steps. gamma[k] is gamma for step k; Adam index t = t0 + k + 1.
 * State arrays are updated in place (p/c/sums hold the state of the current p).
 * Returns 0, or 5 if a non-finite theta appeared (SPEC.md:396 abort). */
int oc_run(int32_t n, const int64_t* rowptr, const int32_t* colidx, const float* wts, const oc_cfg* cf,
           const float* gamma, int64_t n_steps, int64_t t0,
           float* theta, float* m, float* v, float* p, float* c, int64_t* sumD, int64_t* sumD2) {
    const int32_t S = cf->S;
    const size_t NS = (size_t)n * S;
    float* p2 = (float*)malloc(sizeof(float) * (NS ? NS : 1));
    float* c2 = (float*)malloc(sizeof(float) * (n ? n : 1));
    int64_t* d2a = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t* d2b = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    float* Tcol = (float*)malloc(sizeof(float) * (S ? S : 1));
    int bad = 0;
    for (int64_t k = 0; k < n_steps && !bad; ++k) {
        float sc[4];
        oc_step_scalars(cf, t0 + k + 1, gamma[k], sc);
        const int thr = cf->threads > 1 ? cf->threads : 1;
        const int64_t t = t0 + k + 1;
        if (cf->problem == OC_MAXCLIQUE_SPARSE) oc_colsum(n, S, p, Tcol);
        (void)thr;
#pragma omp parallel num_threads(thr) reduction(| : bad)
        {
            float* q = (float*)malloc(sizeof(float) * (S ? S : 1));
#pragma omp for schedule(static)
            for (int32_t i = 0; i < n; ++i) {
                const size_t r = (size_t)i * S;
                bad |= update_row(i, n, t, rowptr, colidx, wts, cf, sc, Tcol, p, theta + r, m + r, v + r,
                                  c[i], sumD[i], sumD2[i], p2 + r, &c2[i], &d2a[i], &d2b[i], q);
            }
            free(q);
        }
        memcpy(p, p2, sizeof(float) * NS);
        memcpy(c, c2, sizeof(float) * n);
        memcpy(sumD, d2a, sizeof(int64_t) * n);
        memcpy(sumD2, d2b, sizeof(int64_t) * n);
    }
    free(p2); free(c2); free(d2a); free(d2b); free(Tcol);
    return bad ? 5 : 0;
}

/* One step for a subset of rows only (sampled checks at full size).
 * Inputs: the full p/c/sums at the start of the step, and theta/m/v of the
 * selected rows ([nrows][S]). Outputs for rows[k]: theta/m/v/p [nrows][S],
 * c/sums [nrows]. */
void oc_step_rows(int32_t n, const int64_t* rowptr, const int32_t* colidx, const float* wts, const oc_cfg* cf,
                  float gamma_t, int64_t t, const float* p, const float* c, const int64_t* sumD,
                  const int64_t* sumD2, const float* theta_rows, const float* m_rows, const float* v_rows,
                  const int32_t* rows, int32_t nrows,
                  float* theta_out, float* m_out, float* v_out, float* p_out,
                  float* c_out, int64_t* sD_out, int64_t* sD2_out) {
    const int32_t S = cf->S;
    float sc[4];
    oc_step_scalars(cf, t, gamma_t, sc);
    float* q = (float*)malloc(sizeof(float) * (S ? S : 1));
    float* Tcol = (float*)malloc(sizeof(float) * (S ? S : 1));
    if (cf->problem == OC_MAXCLIQUE_SPARSE) oc_colsum(n, S, p, Tcol);
    for (int32_t k = 0; k < nrows; ++k) {
        const int32_t i = rows[k];
        const size_t r = (size_t)k * S;
        memcpy(theta_out + r, theta_rows + r, sizeof(float) * S);
        memcpy(m_out + r, m_rows + r, sizeof(float) * S);
        memcpy(v_out + r, v_rows + r, sizeof(float) * S);
        (void)update_row(i, n, t, rowptr, colidx, wts, cf, sc, Tcol, p, theta_out + r, m_out + r, v_out + r,
                   c[i], sumD[i], sumD2[i], p_out + r, &c_out[k], &sD_out[k], &sD2_out[k], q);
    }
    free(q);
    free(Tcol);
}

/* ------------------------------------------------------- evaluation ---- */
/* x = [theta >= thr] (thr = 0 for the sigmoid map, 1/2 for clamp where theta
 * holds p); counts[s][3] = (size, violations, cut) with each
 * undirected edge counted once (j > i); energy[s] = -size + lam*viol
 * (MIS / clique on the complement) or -cut (Max-Cut); *best = argmin energy,
 * lowest index on ties. */
void oc_eval(int32_t n, const int64_t* rowptr, const int32_t* colidx, const float* wts, int32_t problem, float lam,
             int32_t S, const float* theta, float thr, int64_t* counts, int64_t* wsums, double* energy,
             int32_t* best) {
    memset(counts, 0, sizeof(int64_t) * 3 * (size_t)S);
    memset(wsums, 0, sizeof(int64_t) * 2 * (size_t)S);
    for (int32_t i = 0; i < n; ++i) {
        for (int32_t s = 0; s < S; ++s) {
            const int xi = theta[(size_t)i * S + s] >= thr;
            counts[3 * s + 0] += xi;
            for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
                const int32_t j = colidx[e];
                if (j <= i) continue;
                const int xj = theta[(size_t)j * S + s] >= thr;
                counts[3 * s + 1] += xi & xj;
                counts[3 * s + 2] += xi ^ xj;
                const int64_t W = wts ? llrintf(wts[e] * 0x1p24f) : ((int64_t)1 << 24);
                wsums[2 * s + 0] += (xi & xj) ? W : 0;
                wsums[2 * s + 1] += (xi ^ xj) ? W : 0;
            }
        }
    }
    if (problem == OC_MAXCLIQUE_SPARSE)   /* complement counts: pairs in x minus edges in x; size(n-size) - cut */
        for (int32_t s = 0; s < S; ++s) {
            const int64_t sz = counts[3 * s + 0];
            counts[3 * s + 1] = sz * (sz - 1) / 2 - counts[3 * s + 1];
            counts[3 * s + 2] = sz * ((int64_t)n - sz) - counts[3 * s + 2];
        }
    int32_t b = 0;
    for (int32_t s = 0; s < S; ++s) {
        /* weighted graphs: the penalty / cut are weight sums (exact fixed point), else edge counts */
        const double viol = wts ? (double)wsums[2 * s + 0] * 0x1p-24 : (double)counts[3 * s + 1];
        const double cut = wts ? (double)wsums[2 * s + 1] * 0x1p-24 : (double)counts[3 * s + 2];
        energy[s] = (problem == OC_MAXCUT) ? -cut : -(double)counts[3 * s + 0] + (double)lam * viol;
        if (energy[s] < energy[b]) b = s;
    }
    *best = b;
}

/* Multi-instance batch (NEXT-3): rows carry their instance in
 * group_of_row[n] (0..G-1); counts[g][s][3] over the rows of group g and the
 * edges (i < j) leaving them; energy[g][s] as in oc_eval; best[g] = argmin over s
 * of energy[g][s], lowest index on ties. */
void oc_eval_groups(int32_t n, const int64_t* rowptr, const int32_t* colidx, int32_t problem, float lam,
                    int32_t S, const float* theta, float thr, const int32_t* group_of_row, int32_t G,
                    int64_t* counts, double* energy, int32_t* best) {
    memset(counts, 0, sizeof(int64_t) * 3 * (size_t)S * (size_t)G);
    for (int32_t i = 0; i < n; ++i) {
        int64_t* cg = counts + (size_t)group_of_row[i] * 3 * (size_t)S;
        for (int32_t s = 0; s < S; ++s) {
            const int xi = theta[(size_t)i * S + s] >= thr;
            cg[3 * s + 0] += xi;
            for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
                const int32_t j = colidx[e];
                if (j <= i) continue;
                const int xj = theta[(size_t)j * S + s] >= thr;
                cg[3 * s + 1] += xi & xj;
                cg[3 * s + 2] += xi ^ xj;
            }
        }
    }
    for (int32_t g = 0; g < G; ++g) {
        const int64_t* cg = counts + (size_t)g * 3 * (size_t)S;
        double* eg = energy + (size_t)g * S;
        int32_t b = 0;
        for (int32_t s = 0; s < S; ++s) {
            eg[s] = (problem == OC_MAXCUT) ? -(double)cg[3 * s + 2]
                                           : -(double)cg[3 * s + 0] + (double)lam * (double)cg[3 * s + 1];
            if (eg[s] < eg[b]) b = s;
        }
        best[g] = b;
    }
}

/* -------------------------------------------------------- complement --- */
/* Complement of a simple graph (for max clique = MIS on the complement).
 * Pass colidx_out = NULL to get the nnz only. Returns nnz of the complement. */
int64_t oc_complement(int32_t n, const int64_t* rowptr, const int32_t* colidx,
                      int64_t* rowptr_out, int32_t* colidx_out) {
    int64_t nnz = 0;
    char* mark = (char*)calloc((size_t)n ? (size_t)n : 1, 1);
    for (int32_t i = 0; i < n; ++i) {
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) mark[colidx[e]] = 1;
        if (rowptr_out) rowptr_out[i] = nnz;
        for (int32_t j = 0; j < n; ++j) {
            if (j == i || mark[j]) continue;
            if (colidx_out) colidx_out[nnz] = j;
            ++nnz;
        }
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) mark[colidx[e]] = 0;
    }
    if (rowptr_out) rowptr_out[n] = nnz;
    free(mark);
    return nnz;
}

/* ================================================== K-ary (NEXT-4) ====== */
/* Graph colouring with K colours (App. B, map P:672-676, energy
 * P:745-750). Arrays are [n][S][K]; the parameter is P itself (row-stochastic
 * per (i, s)): AdamW on P with dR/dP, (+ noise), then P = Clamp(P') / sum_k
 * Clamp(P'_k) (uniform 1/K if every clamp is 0). Statistics per (i, k) over the
 * replicas, with the binary path's fixed-point contract (shift = previous mean).
 *   dR/dp_isk = q_isk + k_t (K p - 1)^(alpha-1) - a_c (p - mu_ik)/STD_ik,
 *   q_isk = sum_{j in N(i)} p_jsk (CSR order), k_t = -gamma_t c_K alpha K,
 *   c_K = 1/((K-1)((K-1)^(alpha-1) + 1)).
 * fp32 contract for the K-ary parts:
 *   - the entropy factor e = fl(fl(K p) - 1), e^(alpha-1) left to right;
 *   - the normaliser Z = ((c_0 + c_1) + c_2) + ..., p_k = c_k / Z;
 *   - noise: colours pair up, key of (t, i, k, s) = base + ((t n + i) K + k_even) S_total + s;
 *     cos half for even k, sin half for odd k. */

/* k_t for the K-ary entropy, host double -> fp32 */
float oc_kt_K(int32_t K, int32_t alpha, float gamma_t) {
    const double cK = 1.0 / ((double)(K - 1) * (pow((double)(K - 1), (double)(alpha - 1)) + 1.0));
    return (float)(-(double)gamma_t * cK * (double)alpha * (double)K);
}

static void normalize_K(const float* w, int32_t K, float* p) {
    float Z = 0.0f;
    for (int32_t k = 0; k < K; ++k) Z = Z + oc_clamp01(w[k]);
    if (Z > 0.0f) {
        for (int32_t k = 0; k < K; ++k) p[k] = oc_clamp01(w[k]) / Z;
    } else {
        const float u = (float)(1.0 / (double)K);
        for (int32_t k = 0; k < K; ++k) p[k] = u;
    }
}

void oc_normalize_K(const float* w, int32_t K, float* p) { normalize_K(w, K, p); }

/* W_0 = 1/K + U(lo, hi) keyed (seed, i K + k, s) (the sum in double, rounded once), P_0 = normalise(W_0);
 * the first statistics shift is c = 1/K (the centre of the simplex); sums of P_0. */
void oc_init_K(int32_t n, const oc_cfg* cf, int32_t K, float* P, float* m, float* v,
               float* c, int64_t* sumD, int64_t* sumD2) {
    const int32_t S = cf->S;
    const uint64_t base = mix64(cf->seed);
    const double lo = (double)cf->init_lo, hi = (double)cf->init_hi;
    float* w = (float*)malloc(sizeof(float) * (size_t)K);
    const float c0 = (float)(1.0 / (double)K);
    for (int32_t i = 0; i < n; ++i) {
        for (int32_t s = 0; s < S; ++s) {
            for (int32_t k = 0; k < K; ++k) {
                const uint64_t key = base + ((uint64_t)i * (uint64_t)K + (uint64_t)k) * (uint64_t)S + (uint64_t)s;
                const uint64_t kk = mix64(key) >> 40;
                w[k] = (float)(1.0 / (double)K + (lo + (hi - lo) * (double)kk * 0x1p-24));
            }
            const size_t at = ((size_t)i * S + s) * K;
            normalize_K(w, K, P + at);
            for (int32_t k = 0; k < K; ++k) { m[at + k] = 0.0f; v[at + k] = 0.0f; }
        }
        for (int32_t k = 0; k < K; ++k) {
            int64_t a = 0, b = 0;
            for (int32_t s = 0; s < S; ++s) {
                const float d = P[((size_t)i * S + s) * K + k] - c0;
                a += llrintf(d * 0x1p40f);
                const float dd = d * d;
                b += llrintf(dd * 0x1p40f);
            }
            c[(size_t)i * K + k] = c0;
            sumD[(size_t)i * K + k] = a;
            sumD2[(size_t)i * K + k] = b;
        }
    }
    free(w);
}

static int update_row_K(int32_t i, int32_t n, int64_t t, const int64_t* rowptr, const int32_t* colidx,
                        const oc_cfg* cf, int32_t K, float kt, const float* sc, const float* P,
                        float* pp, float* mm, float* vv, const float* c_i, const int64_t* sD_i,
                        const int64_t* sD2_i, float* p_new, float* c_new, int64_t* sD_new, int64_t* sD2_new,
                        float* q, float* w, float* mu, float* sd) {
    const int32_t S = cf->S;
    const float at = sc[1], st = sc[2], rt = sc[3];
    const float b1 = cf->beta1, b2 = cf->beta2, eps = cf->eps;
    const float c1 = (float)(1.0 - (double)cf->beta1), c2 = (float)(1.0 - (double)cf->beta2);
    const float ac = cf->comm, Kf = (float)K;
    const float ns = oc_noise_scale(cf);
    const uint64_t nbase = oc_noise_base(cf->seed);
    int bad = 0;
    for (int32_t k = 0; k < K; ++k) finalize_stats(c_i[k], sD_i[k], sD2_i[k], S, &mu[k], &sd[k]);
    for (int32_t s = 0; s < S; ++s) {
        for (int32_t k = 0; k < K; ++k) q[k] = 0.0f;
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
            const float* pj = P + ((size_t)colidx[e] * S + s) * K;
            for (int32_t k = 0; k < K; ++k) q[k] = q[k] + pj[k];
        }
        const size_t at_s = (size_t)s * K;        /* offset of (s, 0) inside row i */
        for (int32_t k = 0; k < K; ++k) {         /* g_k = dR/dp_k, into q[k] */
            const float pi = pp[at_s + k];
            const float e = Kf * pi - 1.0f;
            float ep = e;
            for (int32_t a = 2; a < cf->alpha; ++a) ep = ep * e;       /* (K p - 1)^(alpha-1) */
            /* Eq. 10 term -alpha_c (p - mu) / STD as (p - mu) kc with the (variable, colour)'s
             * kc = fl(-alpha_c / STD) (0 if STD < 1e-6), as the binary contract (R6) */
            const float kc = (sd[k] >= 1e-6f) ? (-ac) / sd[k] : 0.0f;
            q[k] = fmaf(pi - mu[k], kc, fmaf(kt, ep, q[k]));   /* (q + entropy) + comm, fused */
        }
        if (cf->kary_grad) {                      /* through the map: g - <g, p>, <g, p> in colour order */
            float gb = 0.0f;
            for (int32_t k = 0; k < K; ++k) gb = gb + q[k] * pp[at_s + k];
            for (int32_t k = 0; k < K; ++k) q[k] = q[k] - gb;
        }
        for (int32_t k = 0; k < K; ++k) {
            const float pi = pp[at_s + k];
            const float g = q[k];
            float t1 = pi * at;
            const float m1 = fmaf(b1, mm[at_s + k], c1 * g);
            const float v1 = fmaf(b2, vv[at_s + k], (c2 * g) * g);
            const float den = fmaf(sqrtf(v1), rt, eps);
            t1 = fmaf(-st, m1 / den, t1);
            if (cf->temperature > 0.0f) {   /* colours pair up (k even, k + 1) on one hash */
                const uint64_t key = nbase + (((uint64_t)t * (uint64_t)n + (uint64_t)i) * (uint64_t)K + (uint64_t)(k & ~1))
                                                 * (uint64_t)S + (uint64_t)s;
                float zc, zs;
                oc_gauss_pair_from_hash(mix64(key), &zc, &zs);
                t1 = fmaf(ns, (k & 1) ? zs : zc, t1);
            }
            if (!isfinite(t1)) bad = 1;
            w[k] = t1;
            mm[at_s + k] = m1;
            vv[at_s + k] = v1;
        }
        normalize_K(w, K, p_new + at_s);
    }
    for (int32_t k = 0; k < K; ++k) {
        int64_t a = 0, b = 0;
        for (int32_t s = 0; s < S; ++s) {
            const float d = p_new[(size_t)s * K + k] - mu[k];
            a += llrintf(d * 0x1p40f);
            const float dd = d * d;
            b += llrintf(dd * 0x1p40f);
        }
        c_new[k] = mu[k];
        sD_new[k] = a;
        sD2_new[k] = b;
    }
    return bad;
}

/* n_steps K-ary annealing steps; P/m/v [n][S][K], c/sums [n][K] in place. Returns 0 or 5 (non-finite). */
int oc_run_K(int32_t n, const int64_t* rowptr, const int32_t* colidx, const oc_cfg* cf, int32_t K,
             const float* gamma, int64_t n_steps, int64_t t0, float* P, float* m, float* v,
             float* c, int64_t* sumD, int64_t* sumD2) {
    const int32_t S = cf->S;
    const size_t NSK = (size_t)n * S * K, NK = (size_t)n * K;
    float* P2 = (float*)malloc(sizeof(float) * (NSK ? NSK : 1));
    float* cc = (float*)malloc(sizeof(float) * (NK ? NK : 1));
    int64_t* da = (int64_t*)malloc(sizeof(int64_t) * (NK ? NK : 1));
    int64_t* db = (int64_t*)malloc(sizeof(int64_t) * (NK ? NK : 1));
    int bad = 0;
    for (int64_t k = 0; k < n_steps && !bad; ++k) {
        float sc[4];
        const int64_t t = t0 + k + 1;
        oc_step_scalars(cf, t, gamma[k], sc);
        const float kt = oc_kt_K(K, cf->alpha, gamma[k]);
        const int thr = cf->threads > 1 ? cf->threads : 1;
        (void)thr;
#pragma omp parallel num_threads(thr) reduction(| : bad)
        {
            float* q = (float*)malloc(sizeof(float) * (size_t)K * 4);
            float* w = q + K;
            float* mu = q + 2 * K;
            float* sd = q + 3 * K;
#pragma omp for schedule(static)
            for (int32_t i = 0; i < n; ++i) {
                const size_t r = (size_t)i * S * K, rk = (size_t)i * K;
                bad |= update_row_K(i, n, t, rowptr, colidx, cf, K, kt, sc, P, P + r, m + r, v + r,
                                    c + rk, sumD + rk, sumD2 + rk, P2 + r, cc + rk, da + rk, db + rk, q, w, mu, sd);
            }
            free(q);
        }
        memcpy(P, P2, sizeof(float) * NSK);
        memcpy(c, cc, sizeof(float) * NK);
        memcpy(sumD, da, sizeof(int64_t) * NK);
        memcpy(sumD2, db, sizeof(int64_t) * NK);
    }
    free(P2); free(cc); free(da); free(db);
    return bad ? 5 : 0;
}

/* x_is = argmax_k P (lowest k on ties); counts[s][3] = (0, conflicts, |E| - conflicts) with
 * conflicts = #{(i<j) in E : x_i = x_j}; energy[s] = conflicts; *best = argmin, lowest s on ties;
 * X (optional, [n][S] uint8) receives the colours. */
void oc_eval_K(int32_t n, const int64_t* rowptr, const int32_t* colidx, int32_t S, int32_t K,
               const float* P, uint8_t* X, int64_t* counts, double* energy, int32_t* best) {
    uint8_t* x = X ? X : (uint8_t*)malloc((size_t)n * S + 1);
    for (int32_t i = 0; i < n; ++i)
        for (int32_t s = 0; s < S; ++s) {
            const float* pr = P + ((size_t)i * S + s) * K;
            int32_t b = 0;
            for (int32_t k = 1; k < K; ++k) if (pr[k] > pr[b]) b = k;
            x[(size_t)i * S + s] = (uint8_t)b;
        }
    memset(counts, 0, sizeof(int64_t) * 3 * (size_t)S);
    int64_t edges = 0;
    for (int32_t i = 0; i < n; ++i)
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
            const int32_t j = colidx[e];
            if (j <= i) continue;
            ++edges;
            for (int32_t s = 0; s < S; ++s) counts[3 * s + 1] += x[(size_t)i * S + s] == x[(size_t)j * S + s];
        }
    int32_t b = 0;
    for (int32_t s = 0; s < S; ++s) {
        counts[3 * s + 2] = edges - counts[3 * s + 1];
        energy[s] = (double)counts[3 * s + 1];
        if (energy[s] < energy[b]) b = s;
    }
    *best = b;
    if (!X) free(x);
}
