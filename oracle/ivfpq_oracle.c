/*
 * TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference IVFPQ
 * search path (reference: /root/reference/pkg/src/ivfpq8/).  Used by tests/
 * as a fast bit-exact checker and by bench.py as an optional CPU baseline.
 * Never linked into, or called by, the product library.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (see oracle/Makefile).
 * -ffp-contract=off is essential: the reference computes every fp32 op as a
 * separate numpy ufunc (one rounding each), so no fused multiply-add.
 *
 * Index layout consumed here is the reference's own: list c holds
 * ids[list_off[c] .. list_off[c+1]) and codes row-major [L_c][s]
 * (index.py:27-38), concatenated over c.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { PREC_F32 = 0, PREC_F16 = 1, PREC_E5M3 = 2, PREC_E4M4 = 3 };

static inline uint32_t f2u(float x) { uint32_t u; memcpy(&u, &x, 4); return u; }
static inline float u2f(uint32_t u) { float x; memcpy(&x, &u, 4); return x; }

/* minifloat.py:91-116 encode_array (exponent rebase + mantissa truncation). */
uint8_t orc_fp8_encode(float x, int prec) {
    int m = prec == PREC_E5M3 ? 3 : 4, bias = prec == PREC_E5M3 ? 15 : 7;
    int emax = (1 << (8 - m)) - 1;
    uint32_t b = f2u(x);
    int e = (int)(b >> 23) - 127 + bias;
    uint32_t mant = (b & 0x7FFFFFu) >> (23 - m);
    if (e < 1) return 0;
    if (e > emax) return 0xFF;
    return (uint8_t)(((uint32_t)e << m) | mant);
}

/* minifloat.py:119-133 decode_array. */
float orc_fp8_decode(uint8_t c, int prec) {
    int m = prec == PREC_E5M3 ? 3 : 4, bias = prec == PREC_E5M3 ? 15 : 7;
    uint32_t e = (uint32_t)c >> m, mant = (uint32_t)c & ((1u << m) - 1);
    if (e == 0) return 0.0f;
    return u2f(((e + 127 - bias) << 23) | (mant << (23 - m)));
}

/* minifloat.py:151-164: min(x, 65504) then binary16 round-to-nearest-even.
 * Input is non-negative and finite (squared norms). */
uint16_t orc_f16_encode(float x) {
    if (x > 65504.0f) x = 65504.0f;
    uint32_t b = f2u(x);
    uint32_t e = b >> 23, m = b & 0x7FFFFFu;
    if (e == 0) return 0;                      /* fp32 subnormal < 2^-126: rounds to +0 */
    int he = (int)e - 127 + 15;
    if (he <= 0) {                             /* binary16 subnormal range */
        uint32_t M = m | 0x800000u;
        int shift = 126 - (int)e;              /* value / 2^-24 = M * 2^-shift */
        if (shift > 24) return 0;
        uint32_t r = M >> shift, rem = M & ((1u << shift) - 1), half = 1u << (shift - 1);
        if (rem > half || (rem == half && (r & 1u))) r++;
        return (uint16_t)r;
    }
    uint32_t r = ((uint32_t)he << 10) | (m >> 13), rem = m & 0x1FFFu;
    if (rem > 0x1000u || (rem == 0x1000u && (r & 1u))) r++;
    return (uint16_t)r;
}

/* minifloat.py:167-169. */
float orc_f16_decode(uint16_t h) {
    uint32_t e = (h >> 10) & 0x1F, m = h & 0x3FF;
    if (e == 0) return (float)m * u2f(0x33800000u); /* m * 2^-24, exact */
    return u2f(((e + 112) << 23) | (m << 13));
}

/* datasets.py:166-176 squared_l2_to_all: diff = base - q; acc += diff*diff. */
static void sq_l2_all(const float *base, int n, int d, const float *q, float *out) {
    for (int c = 0; c < n; ++c) {
        float acc = 0.0f;
        const float *row = base + (size_t)c * d;
        for (int t = 0; t < d; ++t) { float df = row[t] - q[t]; float sq = df * df; acc = acc + sq; }
        out[c] = acc;
    }
}

typedef struct { float d; int64_t id; } cand_t;
static int cand_cmp(const void *a, const void *b) {
    const cand_t *x = a, *y = b;
    if (x->d < y->d) return -1;
    if (x->d > y->d) return 1;
    return (x->id > y->id) - (x->id < y->id);
}

/* search.py:91-97 select_clusters: stable argsort of d2, first nprobe. */
void orc_select(const float *coarse, int nlist, int d, const float *q, int nprobe, int64_t *out) {
    float *d2 = malloc(sizeof(float) * nlist);
    cand_t *c = malloc(sizeof(cand_t) * nlist);
    sq_l2_all(coarse, nlist, d, q, d2);
    for (int i = 0; i < nlist; ++i) { c[i].d = d2[i]; c[i].id = i; }
    qsort(c, nlist, sizeof(cand_t), cand_cmp);
    for (int i = 0; i < nprobe; ++i) out[i] = c[i].id;
    free(d2); free(c);
}

/* search.py:100-127 _raw_table + build_lut.  entries: f32 / u16 / u8 per prec. */
void orc_build_lut(const float *centers, int s, int n_codes, int sub_d, const float *rq, int prec, void *entries) {
    for (int j = 0; j < s; ++j)
        for (int m = 0; m < n_codes; ++m) {
            const float *cw = centers + ((size_t)j * n_codes + m) * sub_d;
            float acc = 0.0f;
            for (int t = 0; t < sub_d; ++t) { float df = cw[t] - rq[j * sub_d + t]; float sq = df * df; acc = acc + sq; }
            size_t e = (size_t)j * n_codes + m;
            if (prec == PREC_F32) ((float *)entries)[e] = acc;
            else if (prec == PREC_F16) ((uint16_t *)entries)[e] = orc_f16_encode(acc);
            else ((uint8_t *)entries)[e] = orc_fp8_encode(acc, prec);
        }
}

static float lut_value(const void *entries, size_t e, int prec) {
    if (prec == PREC_F32) return ((const float *)entries)[e];
    if (prec == PREC_F16) return orc_f16_decode(((const uint16_t *)entries)[e]);
    return orc_fp8_decode(((const uint8_t *)entries)[e], prec);
}

/* search.py:130-142 scan_list: R = sum_j decode(T[j][code_j]), sequential j. */
void orc_scan(const uint8_t *codes, int64_t L, int s, int n_codes, const void *entries, int prec, float *out) {
    for (int64_t v = 0; v < L; ++v) {
        float acc = 0.0f;
        for (int j = 0; j < s; ++j) acc = acc + lut_value(entries, (size_t)j * n_codes + codes[v * s + j], prec);
        out[v] = acc;
    }
}

/* search.py:158-203 search + search_batch (padding -1/+inf, short count). */
int64_t orc_search_batch(const float *coarse, int nlist, int d, const float *centers, int s, int p,
                         const int64_t *list_off, const int64_t *ids, const uint8_t *codes,
                         const float *queries, int nq, int k, int nprobe, int prec,
                         int64_t *out_ids, float *out_d, int nthreads) {
    int n_codes = 1 << p, sub_d = d / s;
    int64_t n_short = 0;
    size_t esz = prec == PREC_F32 ? 4 : prec == PREC_F16 ? 2 : 1;
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1) reduction(+ : n_short)
    {
        int64_t *probes = malloc(sizeof(int64_t) * nprobe);
        float *rq = malloc(sizeof(float) * d);
        void *lut = malloc(esz * s * n_codes);
        size_t cap = 1024;
        cand_t *cand = malloc(sizeof(cand_t) * cap);
        float *r = NULL; size_t rcap = 0;
#pragma omp for schedule(dynamic, 4)
        for (int qi = 0; qi < nq; ++qi) {
            const float *q = queries + (size_t)qi * d;
            orc_select(coarse, nlist, d, q, nprobe, probes);
            size_t n = 0;
            for (int pi = 0; pi < nprobe; ++pi) {
                int64_t c = probes[pi], lo = list_off[c], L = list_off[c + 1] - lo;
                if (L == 0) continue;
                for (int t = 0; t < d; ++t) rq[t] = q[t] - coarse[(size_t)c * d + t];
                orc_build_lut(centers, s, n_codes, sub_d, rq, prec, lut);
                if ((size_t)L > rcap) { rcap = L; r = realloc(r, sizeof(float) * rcap); }
                orc_scan(codes + (size_t)lo * s, L, s, n_codes, lut, prec, r);
                if (n + L > cap) { while (n + L > cap) cap *= 2; cand = realloc(cand, sizeof(cand_t) * cap); }
                for (int64_t v = 0; v < L; ++v) { cand[n].d = r[v]; cand[n].id = ids[lo + v]; ++n; }
            }
            qsort(cand, n, sizeof(cand_t), cand_cmp);
            for (int i = 0; i < k; ++i) {
                out_ids[(size_t)qi * k + i] = i < (int64_t)n ? cand[i].id : -1;
                out_d[(size_t)qi * k + i] = i < (int64_t)n ? cand[i].d : INFINITY;
            }
            if ((int64_t)n < k) n_short += 1;
        }
        free(probes); free(rq); free(lut); free(cand); free(r);
    }
    return n_short;
}

/* datasets.py:179-201 brute_force_knn (sequential fp32 distance, ties -> lower id). */
void orc_brute_force_knn(const float *base, int64_t n, int d, const float *queries, int nq, int k,
                         int64_t *out_ids, float *out_d, int nthreads) {
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1)
    {
        float *d2 = malloc(sizeof(float) * n);
        cand_t *c = malloc(sizeof(cand_t) * n);
#pragma omp for schedule(dynamic, 1)
        for (int qi = 0; qi < nq; ++qi) {
            sq_l2_all(base, (int)n, d, queries + (size_t)qi * d, d2);
            for (int64_t i = 0; i < n; ++i) { c[i].d = d2[i]; c[i].id = i; }
            qsort(c, n, sizeof(cand_t), cand_cmp);
            for (int i = 0; i < k; ++i) { out_ids[(size_t)qi * k + i] = c[i].id; out_d[(size_t)qi * k + i] = c[i].d; }
        }
        free(d2); free(c);
    }
}

/* ---- ingest: pq_encode (pq.py:92-110) via assign_to_centroids (kmeans.py:49-69)
 * per subspace, restating the BLAS / einsum arithmetic numpy uses for it
 * (probed in the build container, pinned by tests/golden/pq_encode.npz):
 *   dot  = sequential fmaf chain over t (OpenBLAS sgemm, kmeans.py:61)
 *   norm = einsum("ij,ij->i"): sequential fl(acc + fl(v_t^2)) for n <= 3,
 *          fl(fl(v0^2 + v1^2) + fl(v2^2 + v3^2)) for n = 4 (kmeans.py:58,64)
 *   dist = fl(fl(fl(-2 dot) + cn) + xn), max(dist, 0), first argmin
 *          (kmeans.py:62-67).  Defined for sub_d <= 4 only. */
static float einsum_sq(const float *v, int n) {
    if (n == 4) {
        float a = v[0] * v[0], b = v[1] * v[1], c = v[2] * v[2], e = v[3] * v[3];
        float s0 = a + b, s1 = c + e;
        return s0 + s1;
    }
    float acc = v[0] * v[0];
    for (int t = 1; t < n; ++t) {
        float sq = v[t] * v[t];
        acc = acc + sq;
    }
    return acc;
}

int orc_pq_encode(const float *X, int64_t n, int d, const float *centers, int s, int n_codes, uint8_t *out) {
    int sub = d / s;
    if (sub < 1 || sub > 4 || sub * s != d) return -1;
    float *cn = (float *)malloc(sizeof(float) * (size_t)s * n_codes);
    for (int64_t e = 0; e < (int64_t)s * n_codes; ++e) cn[e] = einsum_sq(centers + e * sub, sub);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        for (int j = 0; j < s; ++j) {
            const float *x = X + i * d + j * sub;
            float xn = einsum_sq(x, sub);
            float best = INFINITY;
            int bi = 0;
            for (int m = 0; m < n_codes; ++m) {
                const float *c = centers + ((int64_t)j * n_codes + m) * sub;
                float dot = 0.0f;
                for (int t = 0; t < sub; ++t) dot = fmaf(x[t], c[t], dot);
                float dist = -2.0f * dot;
                dist = dist + cn[(int64_t)j * n_codes + m];
                dist = dist + xn;
                if (dist < 0.0f) dist = 0.0f;
                if (dist < best) {
                    best = dist;
                    bi = m;
                }
            }
            out[i * s + j] = (uint8_t)bi;
        }
    }
    free(cn);
    return 0;
}
