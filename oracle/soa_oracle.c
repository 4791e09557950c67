/* TEST INFRASTRUCTURE — see soa_oracle.h.  Compiled with -ffp-contract=off so
 * that every multiply and add rounds separately, as the reference's g++ -O2
 * x86-64 build does. */
#define _GNU_SOURCE
#include "soa_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static uint64_t lowmask(int bits) { return bits >= 64 ? ~(uint64_t)0 : (((uint64_t)1 << bits) - 1); }

static uint64_t dbits(double x) { uint64_t b; memcpy(&b, &x, 8); return b; }
static double bitsd(uint64_t b) { double x; memcpy(&x, &b, 8); return x; }

static int top_bit(uint64_t v) { return 63 - __builtin_clzll(v); }

/* fpcodec.cpp:15-24 — shift right with round-half-to-even */
static uint64_t rne_shift(uint64_t sig, int shift) {
    if (shift <= 0) return sig << -shift;
    if (shift > 64) return 0;
    if (shift == 64) return sig > ((uint64_t)1 << 63) ? 1 : 0;
    uint64_t q = sig >> shift, r = sig & lowmask(shift), half = (uint64_t)1 << (shift - 1);
    return (r > half || (r == half && (q & 1))) ? q + 1 : q;
}

/* fpcodec.cpp:28-37 */
int or_layout_for(int t, int* e, int* m) {
    if (t < 7 || t > 64) return -1;
    *e = t >= 33 ? 11 : t >= 17 ? 8 : 5;
    *m = t - 1 - *e;
    return 0;
}

static int base_of(int e) { return e == 11 ? 64 : e == 8 ? 32 : 16; }

int or_fmt_width(int fmt) {
    int e, m;
    if (fmt == OR_I64) return 64;
    if (fmt == OR_BF16) return 16;
    if (fmt >= 1000) { or_layout_for(fmt - 1000, &e, &m); return base_of(e); }
    return fmt;
}

/* fpcodec.cpp:39-90 — RNE to IEEE(e, m); overflow -> inf; subnormal targets;
 * NaN keeps the top payload bits and never collapses to infinity. */
uint64_t or_narrow_to_ieee(double x, int e, int m) {
    uint64_t src = dbits(x);
    if (e == 11 && m == 52) return src;
    uint64_t sign = (src >> 63) << (e + m);
    int sexp = (int)((src >> 52) & 0x7ff);
    uint64_t sman = src & lowmask(52);
    int bias = (1 << (e - 1)) - 1, emax = (1 << e) - 1;
    uint64_t inf = sign | ((uint64_t)emax << m);
    if (sexp == 0x7ff) {
        if (sman == 0) return inf;
        uint64_t pay = sman >> (52 - m);
        return inf | (pay ? pay : (uint64_t)1 << (m - 1));
    }
    uint64_t sig;
    int unb;
    if (sexp == 0) {
        if (sman == 0) return sign;
        int lead = top_bit(sman);
        sig = sman << (52 - lead);
        unb = -1022 - (52 - lead);
    } else {
        sig = ((uint64_t)1 << 52) | sman;
        unb = sexp - 1023;
    }
    int texp = unb + bias;
    if (texp >= emax) return inf;
    if (texp >= 1) {
        uint64_t r = rne_shift(sig, 52 - m);
        if (r >> (m + 1)) {
            r >>= 1;
            if (++texp >= emax) return inf;
        }
        return sign | ((uint64_t)texp << m) | (r & lowmask(m));
    }
    return sign | rne_shift(sig, (52 - m) + (1 - texp));
}

/* fpcodec.cpp:92-117 — exact widening to binary64 */
double or_widen_from_ieee(uint64_t b, int e, int m) {
    if (e == 11 && m == 52) return bitsd(b);
    uint64_t s = (b >> (e + m)) & 1;
    int ex = (int)((b >> m) & lowmask(e));
    uint64_t man = b & lowmask(m);
    int bias = (1 << (e - 1)) - 1, emax = (1 << e) - 1;
    uint64_t out;
    if (ex == emax) {
        out = (s << 63) | ((uint64_t)0x7ff << 52) | (man << (52 - m));
    } else if (ex == 0) {
        if (man == 0) {
            out = s << 63;
        } else {
            int lead = top_bit(man);
            int unb = (1 - bias) - m + lead;
            out = (s << 63) | ((uint64_t)(unb + 1023) << 52) | ((man << (52 - lead)) & lowmask(52));
        }
    } else {
        out = (s << 63) | ((uint64_t)(ex - bias + 1023) << 52) | (man << (52 - m));
    }
    return bitsd(out);
}

/* fpcodec.cpp:119-124 */
uint64_t or_expand_to_base_bits(uint64_t bits, int t) {
    int e, m;
    or_layout_for(t, &e, &m);
    int bm = base_of(e) - 1 - e;
    return ((bits >> m) << bm) | ((bits & lowmask(m)) << (bm - m));
}

/* fpcodec.cpp:126-135 — drop mantissa bits toward zero, NaN guard */
uint64_t or_truncate_from_base_bits(uint64_t base, int t) {
    int e, m;
    or_layout_for(t, &e, &m);
    int bm = base_of(e) - 1 - e;
    uint64_t se = base >> bm, full = base & lowmask(bm), man = full >> (bm - m);
    if ((se & lowmask(e)) == lowmask(e) && full != 0 && man == 0) man = (uint64_t)1 << (m - 1);
    return (se << m) | man;
}

/* fpcodec.cpp:137-155 */
uint64_t or_encode_bits(double x, int t) {
    int e, m;
    or_layout_for(t, &e, &m);
    return or_truncate_from_base_bits(or_narrow_to_ieee(x, e, base_of(e) - 1 - e), t);
}
double or_decode_bits(uint64_t b, int t) {
    int e, m;
    or_layout_for(t, &e, &m);
    return or_widen_from_ieee(or_expand_to_base_bits(b, t), e, base_of(e) - 1 - e);
}
double or_quantize(double x, int t) { return or_decode_bits(or_encode_bits(x, t), t); }

/* BufferView::set / get (sph.cpp:103-126) per storage format */
uint64_t or_encode_fmt(double x, int fmt) {
    if (fmt == OR_BF16) return or_narrow_to_ieee(x, 8, 7);
    if (fmt == OR_I64) return (uint64_t)(int64_t)x;
    if (fmt >= 1000) return or_expand_to_base_bits(or_encode_bits(x, fmt - 1000), fmt - 1000);
    return or_encode_bits(x, fmt);
}
double or_decode_fmt(uint64_t b, int fmt) {
    int e, m;
    if (fmt == OR_BF16) return or_widen_from_ieee(b, 8, 7);
    if (fmt == OR_I64) return (double)(int64_t)b;
    if (fmt >= 1000) {
        or_layout_for(fmt - 1000, &e, &m);
        return or_widen_from_ieee(b, e, base_of(e) - 1 - e);
    }
    return or_decode_bits(b, fmt);
}
void or_encode_array(const double* x, uint64_t n, int fmt, uint64_t* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = or_encode_fmt(x[i], fmt);
}
void or_decode_array(const uint64_t* b, uint64_t n, int fmt, double* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = or_decode_fmt(b[i], fmt);
}

/* bitpack.cpp:23-58 — little-endian bit stream, bit k -> byte k>>3, bit k&7.
 * Restated bit-by-bit (the reference's oracles.hpp:18-40 style). */
void or_write_bits(uint8_t* buf, uint64_t off, int w, uint64_t v) {
    for (int k = 0; k < w; ++k) {
        uint64_t bit = off + k;
        uint8_t mask = (uint8_t)(1u << (bit & 7));
        if ((v >> k) & 1) buf[bit >> 3] |= mask;
        else buf[bit >> 3] &= (uint8_t)~mask;
    }
}
uint64_t or_read_bits(const uint8_t* buf, uint64_t off, int w) {
    uint64_t v = 0;
    for (int k = 0; k < w; ++k) {
        uint64_t bit = off + k;
        v |= (uint64_t)((buf[bit >> 3] >> (bit & 7)) & 1) << k;
    }
    return v;
}

void or_apply_moves(const uint8_t* src, uint8_t* dst, uint64_t count, const or_move* mv,
                    int nmoves) {
    for (int f = 0; f < nmoves; ++f) {
        const or_move* p = &mv[f];
        int sw = or_fmt_width(p->src_fmt), dw = or_fmt_width(p->dst_fmt);
        for (uint64_t r = 0; r < count; ++r)
            for (int l = 0; l < p->arity; ++l) {
                uint64_t v = or_read_bits(src, p->src_base + r * p->src_stride + (uint64_t)l * sw, sw);
                if (p->src_fmt != p->dst_fmt) {
                    if (p->src_fmt == OR_I64 || p->dst_fmt == OR_I64) v = v;  /* ints: raw */
                    else v = or_encode_fmt(or_decode_fmt(v, p->src_fmt), p->dst_fmt);
                }
                or_write_bits(dst, p->dst_base + r * p->dst_stride + (uint64_t)l * dw, dw, v);
            }
    }
}

/* pipelines.cpp:51-60 — FNV-1a 64 over the bytes, then length_bits LE */
uint64_t or_checksum(const uint8_t* bytes, uint64_t n, uint64_t length_bits) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t i = 0; i < n; ++i) { h ^= bytes[i]; h *= 0x100000001b3ull; }
    for (int i = 0; i < 8; ++i) { h ^= (uint8_t)(length_bits >> (8 * i)); h *= 0x100000001b3ull; }
    return h;
}

/* sph.cpp:17-24: M4 cubic spline, sigma = 1/pi, support 2h.  Same
 * association order as the C++ source (left to right). */
double or_w(double r, double h) {
    double q = r / h;
    if (q >= 2.0) return 0.0;
    double norm = (1.0 / 3.14159265358979323846) / (h * h * h);
    if (q < 1.0) return norm * (1.0 - 1.5 * q * q + 0.75 * q * q * q);
    double t = 2.0 - q;
    return norm * 0.25 * t * t * t;
}

static double pair_term(const double* x, const double* m, const double* h, uint64_t i, uint64_t j) {
    double dx0 = x[3 * i] - x[3 * j], dx1 = x[3 * i + 1] - x[3 * j + 1], dx2 = x[3 * i + 2] - x[3 * j + 2];
    double r = sqrt(dx0 * dx0 + dx1 * dx1 + dx2 * dx2);
    double hij = 0.5 * (h[i] + h[j]);
    return m[j] * or_w(r, hij);
}

/* sph.cpp:176-199 (density_kernel) over sph.cpp:286-308 chunks */
void or_density_buffer(const double* x, const double* m, const double* h, uint64_t n,
                       uint64_t bs, int rho_fmt, double* rho) {
    for (uint64_t b = 0; b < n; b += bs)
        for (uint64_t i = b; i < b + bs && i < n; ++i) {
            double acc = 0.0;
            for (uint64_t j = b; j < b + bs && j < n; ++j) {
                acc += pair_term(x, m, h, i, j);
                if (rho_fmt) acc = or_decode_fmt(or_encode_fmt(acc, rho_fmt), rho_fmt);
            }
            rho[i] = acc;
        }
}

static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}

/* Cell list of a cubic grid [lo, hi)^3 with cells of side `cell` (particles
 * outside clamp to the face cells), each cell's members in ascending index. */
typedef struct {
    int nc;
    uint64_t *start, *idx;
    int* cid;
} CellList;

static CellList cells_build(const double* x, uint64_t n, double lo, double hi, double cell) {
    CellList L;
    L.nc = (int)ceil((hi - lo) / cell);
    if (L.nc < 1) L.nc = 1;
    const int nc = L.nc;
    uint64_t ncell = (uint64_t)nc * nc * nc;
    L.start = calloc(ncell + 1, sizeof(uint64_t));
    L.idx = malloc((n ? n : 1) * sizeof(uint64_t));
    L.cid = malloc((n ? n : 1) * sizeof(int) * 3);
    for (uint64_t i = 0; i < n; ++i)
        for (int d = 0; d < 3; ++d) {
            int c = (int)floor((x[3 * i + d] - lo) / cell);
            L.cid[3 * i + d] = c < 0 ? 0 : c >= nc ? nc - 1 : c;
        }
    for (uint64_t i = 0; i < n; ++i)
        L.start[((uint64_t)L.cid[3 * i] * nc + L.cid[3 * i + 1]) * nc + L.cid[3 * i + 2] + 1]++;
    for (uint64_t c = 0; c < ncell; ++c) L.start[c + 1] += L.start[c];
    uint64_t* fill = malloc(ncell * sizeof(uint64_t));
    memcpy(fill, L.start, ncell * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i)  /* ascending i -> each cell list is sorted */
        L.idx[fill[((uint64_t)L.cid[3 * i] * nc + L.cid[3 * i + 1]) * nc + L.cid[3 * i + 2]]++] = i;
    free(fill);
    return L;
}

static void cells_free(CellList* L) { free(L->start); free(L->idx); free(L->cid); }

/* the members of the 27 cells around particle i, ascending index */
static uint64_t cells_candidates(const CellList* L, uint64_t i, uint64_t** cand, uint64_t* cap) {
    const int nc = L->nc;
    uint64_t nn = 0;
    for (int a = -1; a <= 1; ++a)
        for (int b = -1; b <= 1; ++b)
            for (int c = -1; c <= 1; ++c) {
                int p = L->cid[3 * i] + a, q = L->cid[3 * i + 1] + b, s = L->cid[3 * i + 2] + c;
                if (p < 0 || q < 0 || s < 0 || p >= nc || q >= nc || s >= nc) continue;
                uint64_t k = ((uint64_t)p * nc + q) * nc + s;
                for (uint64_t t = L->start[k]; t < L->start[k + 1]; ++t) {
                    if (nn == *cap) { *cap *= 2; *cand = realloc(*cand, *cap * sizeof(uint64_t)); }
                    (*cand)[nn++] = L->idx[t];
                }
            }
    qsort(*cand, nn, sizeof(uint64_t), cmp_u64);
    return nn;
}

/* Cell-linked density: density_kernel's sum (sph.cpp:176-199) over every
 * particle of the 27 cells (side >= 2 h_max) in ascending index — the terms
 * beyond the support are exactly +0.0, so this equals the all-pairs sum. */
static double density_home(const CellList* L, const double* x, const double* m, const double* h, uint64_t i,
                           uint64_t** cand, uint64_t* cap) {
    uint64_t nn = cells_candidates(L, i, cand, cap);
    double acc = 0.0;
    for (uint64_t t = 0; t < nn; ++t) acc += pair_term(x, m, h, i, (*cand)[t]);
    return acc;
}

void or_density_cells(const double* x, const double* m, const double* h, uint64_t n,
                      double lo, double hi, double cell, double* rho) {
    CellList L = cells_build(x, n, lo, hi, cell);
    uint64_t cap = 1024, *cand = malloc(cap * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) rho[i] = density_home(&L, x, m, h, i, &cand, &cap);
    free(cand);
    cells_free(&L);
}

/* The same sum for the listed homes only (every particle stays a candidate):
 * the parity check of a large population on a sample of homes. */
void or_density_cells_at(const double* x, const double* m, const double* h, uint64_t n, double lo, double hi,
                         double cell, const uint64_t* homes, uint64_t nh, double* rho) {
    CellList L = cells_build(x, n, lo, hi, cell);
    uint64_t cap = 1024, *cand = malloc(cap * sizeof(uint64_t));
    for (uint64_t k = 0; k < nh; ++k) rho[k] = density_home(&L, x, m, h, homes[k], &cand, &cap);
    free(cand);
    cells_free(&L);
}

/* sph.cpp:26-33 */
double or_dw_dr(double r, double h) {
    double q = r / h;
    if (q >= 2.0) return 0.0;
    double norm = (1.0 / 3.14159265358979323846) / (h * h * h * h);
    if (q < 1.0) return norm * (-3.0 * q + 2.25 * q * q);
    double t = 2.0 - q;
    return norm * (-0.75 * t * t);
}

/* Cell-linked force: force_kernel (sph.cpp:201-245, Deferred writeback) over
 * the 27-cell candidates in ascending index, j == i skipped, grad_w
 * (sph.cpp:35-40) zero at r == 0.  a[3n] and du[n] as the reference writes
 * them; a_scale[n] = sum_j |m_j pf_ij grad W_ij| and du_scale[n] =
 * |P_i/rho_i^2| sum_j |m_j (v_i - v_j) . grad W_ij| are the magnitudes the
 * sums cancel from (the scale a floating-point tolerance is relative to).
 * Returns -1 when some rho is 0 (the reference's domain_error), else 0. */
static void force_home(const CellList* L, const double* x, const double* v, const double* m, const double* h,
                       const double* rho, const double* P, uint64_t i, uint64_t** cand, uint64_t* cap, double* a,
                       double* du, double* a_scale, double* du_scale) {
    uint64_t nn = cells_candidates(L, i, cand, cap);
    const double pi = P[i] / (rho[i] * rho[i]);
    double acc[3] = {0.0, 0.0, 0.0}, compr = 0.0, sa = 0.0, sd = 0.0;
    for (uint64_t t = 0; t < nn; ++t) {
        const uint64_t j = (*cand)[t];
        if (j == i) continue;
        const double d0 = x[3 * i] - x[3 * j], d1 = x[3 * i + 1] - x[3 * j + 1], d2 = x[3 * i + 2] - x[3 * j + 2];
        const double hij = 0.5 * (h[i] + h[j]);
        const double r = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
        double g0 = 0.0, g1 = 0.0, g2 = 0.0;
        if (r != 0.0) {
            const double sc = or_dw_dr(r, hij) / r;
            g0 = sc * d0; g1 = sc * d1; g2 = sc * d2;
        }
        const double pf = pi + P[j] / (rho[j] * rho[j]);
        acc[0] -= m[j] * pf * g0;
        acc[1] -= m[j] * pf * g1;
        acc[2] -= m[j] * pf * g2;
        const double dv = (v[3 * i] - v[3 * j]) * g0 + (v[3 * i + 1] - v[3 * j + 1]) * g1 +
                          (v[3 * i + 2] - v[3 * j + 2]) * g2;
        compr += m[j] * dv;
        sa += fabs(m[j] * pf) * sqrt(g0 * g0 + g1 * g1 + g2 * g2);
        sd += fabs(m[j] * dv);
    }
    for (int l = 0; l < 3; ++l) a[l] = acc[l];
    *du = pi * compr;
    *a_scale = sa;
    *du_scale = fabs(pi) * sd;
}

int or_force_cells(const double* x, const double* v, const double* m, const double* h, const double* rho,
                   const double* P, uint64_t n, double lo, double hi, double cell, double* a, double* du,
                   double* a_scale, double* du_scale) {
    for (uint64_t i = 0; i < n; ++i)
        if (rho[i] == 0.0) return -1;
    CellList L = cells_build(x, n, lo, hi, cell);
    uint64_t cap = 1024, *cand = malloc(cap * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i)
        force_home(&L, x, v, m, h, rho, P, i, &cand, &cap, a + 3 * i, du + i, a_scale + i, du_scale + i);
    free(cand);
    cells_free(&L);
    return 0;
}

/* or_force_cells for the listed homes only (outputs indexed by list slot). */
int or_force_cells_at(const double* x, const double* v, const double* m, const double* h, const double* rho,
                      const double* P, uint64_t n, double lo, double hi, double cell, const uint64_t* homes,
                      uint64_t nh, double* a, double* du, double* a_scale, double* du_scale) {
    for (uint64_t i = 0; i < n; ++i)
        if (rho[i] == 0.0) return -1;
    CellList L = cells_build(x, n, lo, hi, cell);
    uint64_t cap = 1024, *cand = malloc(cap * sizeof(uint64_t));
    for (uint64_t k = 0; k < nh; ++k)
        force_home(&L, x, v, m, h, rho, P, homes[k], &cand, &cap, a + 3 * k, du + k, a_scale + k, du_scale + k);
    free(cand);
    cells_free(&L);
    return 0;
}

/* ---- std::mt19937_64 (the C++ standard's parameters) -------------------- */
typedef struct { uint64_t mt[312]; int i; } mt64;
static void mt_seed(mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->i = 312;
}
static uint64_t mt_next(mt64* s) {
    if (s->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            uint64_t y = (s->mt[k] & 0xFFFFFFFF80000000ull) | (s->mt[(k + 1) % 312] & 0x7FFFFFFFull);
            s->mt[k] = s->mt[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ull : 0);
        }
        s->i = 0;
    }
    uint64_t x = s->mt[s->i++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}
/* libstdc++ generate_canonical<double,53> with one 64-bit draw, then
 * uniform_real_distribution: u * (b - a) + a */
static double mt_uniform(mt64* s, double a, double b) {
    double u = (double)mt_next(s) / 18446744073709551616.0;
    if (u >= 1.0) u = nextafter(1.0, 0.0);
    return u * (b - a) + a;
}

/* sph.cpp:325-349 + sph.cpp:42-46 (eos) */
void or_random_ics(uint64_t n, uint64_t seed, uint64_t accel_seed, double dt, double* x,
                   double* v, double* a, double* u, double* m, double* h, double* rho,
                   double* P, double* cs, double* du, double* dtf, int64_t* id) {
    mt64 rng;
    mt_seed(&rng, seed);
    const double gamma = 5.0 / 3.0;
    for (uint64_t i = 0; i < n; ++i) {
        for (int l = 0; l < 3; ++l) x[3 * i + l] = mt_uniform(&rng, 0.0, 1.0);
        for (int l = 0; l < 3; ++l) v[3 * i + l] = mt_uniform(&rng, -1.0, 1.0);
        u[i] = mt_uniform(&rng, 0.5, 1.5);
        m[i] = 1.0 / 64;
        h[i] = 0.5;
        rho[i] = 1.0;
        P[i] = (gamma - 1.0) * rho[i] * u[i];
        cs[i] = sqrt(gamma * P[i] / rho[i]);
        a[3 * i] = a[3 * i + 1] = a[3 * i + 2] = 0.0;
        du[i] = 0.0;
        dtf[i] = dt;
        id[i] = (int64_t)i;
    }
    if (accel_seed) {
        mt64 r2;
        mt_seed(&r2, accel_seed);
        for (uint64_t i = 0; i < n; ++i) {
            for (int l = 0; l < 3; ++l) a[3 * i + l] = mt_uniform(&r2, -1.0, 1.0);
            du[i] = mt_uniform(&r2, -1.0, 1.0);
        }
    }
}
