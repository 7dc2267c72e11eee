/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously correct CPU implementation of what the B200 path
 * computes (arxiv 2405.02256, "eucalc"). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2405_02256_b200/csrc); neither includes the other.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n.
 * Readings of the paper where it is wrong or silent are those of SURVEY.md §8(c)
 * (E1..E19), listed again in DESIGN.md.
 *
 * Everything is int64 for weights/sums (phi takes integer values;
 * E17) and long double for the hybrid transform.
 *
 * Layout: an image is row-major (last axis fastest); a doubled grid cell
 * u has dim = #odd u_i; vertex p <-> u = 2p.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define EO_MAXN 4
enum { EO_VERTEX = 0, EO_TOP = 1 };
enum { EO_GAUSS = 0, EO_COS = 1, EO_SIN = 2, EO_EXP = 3, EO_ONE = 4 };

static void unrank(int64_t k, int n, const int64_t *d, int64_t *u) {
    for (int i = n - 1; i >= 0; --i) { u[i] = k % d[i]; k /= d[i]; }
}

static int64_t rank_of(int n, const int64_t *d, const int64_t *u) {
    int64_t k = 0;
    for (int i = 0; i < n; ++i) k = k * d[i] + u[i];
    return k;
}

/* ---------------------------------------------------------------------------
 * Step 1: the weighted cubical complex on the doubled grid.
 *
 * EO_TOP: "one top-dimensional cell is associated to each pixel and
 *           the values of lower-dimensional cells are equal to the minimum of
 *           the values of their cofaces"; d_i = 2 m_i + 1. Top cell of
 *           pixel p sits at u = 2p+1; a cell's top cofaces are the pixels q with
 *           q_i = (u_i-1)/2 if u_i odd, q_i in {u_i/2 - 1, u_i/2} if u_i even
 *           (those inside the image). phi(u) = min over them.
 * EO_VERTEX: "initializing the values of the vertices with the pixel
 *           values ... higher-dimensional cells as the minimum of the values of
 *           their vertices"; d_i = 2 m_i - 1.
 * cells: int32 [prod d_i]. Returns 0, or -1 on bad arguments.
 * ------------------------------------------------------------------------- */
int eo_doubled_grid(const int32_t *img, int n, const int64_t *m, int construction,
                    int32_t *cells)
{
    if (n < 1 || n > EO_MAXN) return -1;
    int64_t d[EO_MAXN], ncell = 1;
    for (int i = 0; i < n; ++i) {
        if (m[i] < 1) return -1;
        d[i] = construction == EO_VERTEX ? 2 * m[i] - 1 : 2 * m[i] + 1;
        ncell *= d[i];
    }
    for (int64_t k = 0; k < ncell; ++k) {
        int64_t u[EO_MAXN];
        unrank(k, n, d, u);
        int64_t best = INT64_MAX;
        /* enumerate up to 2 choices per axis */
        for (int mask = 0; mask < (1 << n); ++mask) {
            int64_t q[EO_MAXN];
            int ok = 1;
            for (int i = 0; i < n; ++i) {
                int bit = (mask >> i) & 1;
                if (construction == EO_VERTEX) {
                    /* vertices of the cell: u_i even -> u_i/2; odd -> (u_i-1)/2, (u_i+1)/2 */
                    q[i] = (u[i] % 2 == 0) ? u[i] / 2 : (u[i] - 1) / 2 + bit;
                } else {
                    /* top cofaces: u_i odd -> (u_i-1)/2; even -> u_i/2 - 1 + bit */
                    q[i] = (u[i] % 2 == 1) ? (u[i] - 1) / 2 : u[i] / 2 - 1 + bit;
                    if (q[i] < 0 || q[i] >= m[i]) ok = 0;
                }
            }
            if (!ok) continue;
            int64_t v = img[rank_of(n, m, q)];
            if (v < best) best = v;
        }
        cells[k] = (int32_t)best; /* every TOP cell has >= 1 top coface since m_i >= 1 */
    }
    return 0;
}

/* Euler characteristic chi(phi) = sum_P (-1)^dim(P) phi(P). */
int64_t eo_euler(const int32_t *cells, int n, const int64_t *d)
{
    int64_t ncell = 1, chi = 0;
    for (int i = 0; i < n; ++i) ncell *= d[i];
    for (int64_t k = 0; k < ncell; ++k) {
        int64_t u[EO_MAXN];
        unrank(k, n, d, u);
        int dim = 0;
        for (int i = 0; i < n; ++i) dim += (int)(u[i] & 1);
        chi += (dim & 1) ? -(int64_t)cells[k] : (int64_t)cells[k];
    }
    return chi;
}

/* ---------------------------------------------------------------------------
 * Step 9: critical tables straight from the star definition.
 *
 * Lower star of vertex x w.r.t. xi: the cofaces Q of x with
 * max_Q xi = xi(x). For an axis-aligned cube these are the cells at doubled
 * coordinates u - delta o eps, delta in {0,1}^n ("we explore all cells
 * with coordinates (4 - delta_0 eps_0, 4 - delta_1 eps_1)"); the upper star uses
 * u + delta o eps. Out-of-range cells do not exist (truncated stars, E16).
 *   dminus[x] = chi(phi|lwst(eps, x))   (classical value)
 *   eplus[x]  = chi(phi|upst(eps, x))   (P:87 ingredient)
 * The TRUE right-minus-left Radon jump is J = dminus - eplus (E1: the paper's
 * printed Delta^ord = eplus - dminus has the wrong sign).
 * e: orthant index, bit i set iff eps_i = +1.
 * ------------------------------------------------------------------------- */
int eo_critical(const int32_t *cells, int n, const int64_t *d, int e,
                int64_t *dminus, int64_t *eplus)
{
    int64_t M[EO_MAXN], nv = 1;
    for (int i = 0; i < n; ++i) { M[i] = (d[i] + 1) / 2; nv *= M[i]; }
    int eps[EO_MAXN];
    for (int i = 0; i < n; ++i) eps[i] = ((e >> i) & 1) ? 1 : -1;
    for (int64_t v = 0; v < nv; ++v) {
        int64_t p[EO_MAXN];
        unrank(v, n, M, p);
        int64_t lo = 0, up = 0;
        for (int delta = 0; delta < (1 << n); ++delta) {
            int64_t ul[EO_MAXN], uu[EO_MAXN];
            int okl = 1, oku = 1, pop = 0;
            for (int i = 0; i < n; ++i) {
                int b = (delta >> i) & 1;
                pop += b;
                ul[i] = 2 * p[i] - b * eps[i];
                uu[i] = 2 * p[i] + b * eps[i];
                if (ul[i] < 0 || ul[i] >= d[i]) okl = 0;
                if (uu[i] < 0 || uu[i] >= d[i]) oku = 0;
            }
            int64_t sgn = (pop & 1) ? -1 : 1;
            if (okl) lo += sgn * cells[rank_of(n, d, ul)];
            if (oku) up += sgn * cells[rank_of(n, d, uu)];
        }
        dminus[v] = lo;
        eplus[v] = up;
    }
    return 0;
}

/* Height range of a cell along the (already axis-scaled) integer direction xs:
 * the cell's vertex coordinates along axis i are floor(u_i/2) .. ceil(u_i/2). */
static void cell_hrange(int n, const int64_t *u, const int64_t *xs, int64_t *hmin, int64_t *hmax)
{
    int64_t a = 0, b = 0;
    for (int i = 0; i < n; ++i) {
        int64_t lo = u[i] / 2, hi = (u[i] + 1) / 2;
        int64_t x0 = xs[i] * lo, x1 = xs[i] * hi;
        a += x0 < x1 ? x0 : x1;
        b += x0 < x1 ? x1 : x0;
    }
    *hmin = a;
    *hmax = b;
}

/* ---------------------------------------------------------------------------
 * Literal tier (tiny inputs): the transforms at one threshold by a full scan of
 * the cells. Heights are integer "lattice heights" H = sum_i xs_i p_i where
 * xs_i = xi_i * L/(M_i - 1) (E10: t = H/L - sum xi_i/2 is strictly increasing in
 * H, so orders, ties and all values are those of the paper's normalised
 * embedding). The threshold is t2 = 2H in doubled units so that the
 * open intervals between lattice heights can be probed at odd t2.
 *
 * ECT(xi, t) = chi[phi_{xi<=t}]. A cell P meets {xi <= t} in
 *   - nothing if min_P > t, a single vertex (weight 0 for 1_P) if min_P = t,
 *   - P with its faces if max_P <= t: contribution (-1)^dim phi(P),
 *   - otherwise a truncated cell plus its cut face, both weighted phi(P):
 *     (-1)^dim + (-1)^(dim-1) = 0.
 * so ECT(t) = sum_{P: max_P xi <= t} (-1)^dim phi(P) (E2 corrects Lemma 1).
 *
 * Radon(xi, t) = chi[phi_{xi=t}] = sum_P phi(P) Radon[1_P](t) by
 * linearity, with Radon[1_x] = 1_{xi(x)} for a vertex and
 * Radon[1_P] = (-1)^(dim P - 1) 1_(min_P xi, max_P xi) otherwise (Lemma 4).
 * ------------------------------------------------------------------------- */
int64_t eo_ect_at(const int32_t *cells, int n, const int64_t *d, const int64_t *xs, int64_t t2)
{
    int64_t ncell = 1, s = 0;
    for (int i = 0; i < n; ++i) ncell *= d[i];
    for (int64_t k = 0; k < ncell; ++k) {
        int64_t u[EO_MAXN], hmin, hmax;
        unrank(k, n, d, u);
        cell_hrange(n, u, xs, &hmin, &hmax);
        int dim = 0;
        for (int i = 0; i < n; ++i) dim += (int)(u[i] & 1);
        if (2 * hmax <= t2) s += (dim & 1) ? -(int64_t)cells[k] : (int64_t)cells[k];
    }
    return s;
}

int64_t eo_radon_at(const int32_t *cells, int n, const int64_t *d, const int64_t *xs, int64_t t2)
{
    int64_t ncell = 1, s = 0;
    for (int i = 0; i < n; ++i) ncell *= d[i];
    for (int64_t k = 0; k < ncell; ++k) {
        int64_t u[EO_MAXN], hmin, hmax;
        unrank(k, n, d, u);
        cell_hrange(n, u, xs, &hmin, &hmax);
        int dim = 0;
        for (int i = 0; i < n; ++i) dim += (int)(u[i] & 1);
        if (dim == 0) {
            if (2 * hmin == t2) s += cells[k];
        } else if (2 * hmin < t2 && t2 < 2 * hmax) {
            s += (dim & 1) ? (int64_t)cells[k] : -(int64_t)cells[k]; /* (-1)^(dim-1) */
        }
    }
    return s;
}

/* ---------------------------------------------------------------------------
 * Swept tier: the same two sums evaluated at every lattice height at once.
 * Per cell, (-1)^dim phi is bucketed at max_P (ECT) and (-1)^(dim-1) phi is
 * added on the open doubled-unit interval (2 min_P, 2 max_P) (Radon); vertices
 * add phi at 2 xi(x). Prefix sums give the functions at every doubled height
 * 2H and every open interval midpoint 2H+1. O(#cells + R) per direction.
 *
 * Canonical (unique, minimal) exact representations:
 *   ECT   : T = heights where ECT changes, E = value from there on (E[0]=0 implicit, E9).
 *   Radon : prev = 0; for each height h ascending: at = R(h), after = R((h, h+1));
 *           at != prev    -> (T_c, E_c) gets (h, at)
 *           after != prev -> (T_o, E')  gets (h, after);  prev = after.
 * Zero-net merged entries are dropped (E8). Any of the output triples may be
 * NULL. Returns 0, -1 on bad args, -2 if an output would exceed cap
 * (the counts are still set to the required sizes), -3 on allocation failure.
 * ------------------------------------------------------------------------- */
int eo_transforms(const int32_t *cells, int n, const int64_t *d, const int64_t *xs,
                  int64_t cap,
                  int64_t *T, int64_t *E, int64_t *nT,
                  int64_t *To, int64_t *Eo, int64_t *nTo,
                  int64_t *Tc, int64_t *Ec, int64_t *nTc)
{
    if (n < 1 || n > EO_MAXN) return -1;
    int64_t ncell = 1, hlo = 0, hhi = 0;
    for (int i = 0; i < n; ++i) {
        ncell *= d[i];
        int64_t ext = xs[i] * ((d[i] - 1) / 2);
        if (ext < 0) hlo += ext; else hhi += ext;
    }
    int64_t R = hhi - hlo + 1;
    int64_t *ect = calloc((size_t)R + 1, sizeof(int64_t));
    int64_t *rv = calloc((size_t)(2 * R + 1), sizeof(int64_t));
    int64_t *rd = calloc((size_t)(2 * R + 2), sizeof(int64_t));
    if (!ect || !rv || !rd) { free(ect); free(rv); free(rd); return -3; }
    for (int64_t k = 0; k < ncell; ++k) {
        int64_t u[EO_MAXN], hmin, hmax;
        unrank(k, n, d, u);
        cell_hrange(n, u, xs, &hmin, &hmax);
        int dim = 0;
        for (int i = 0; i < n; ++i) dim += (int)(u[i] & 1);
        int64_t w = cells[k];
        ect[hmax - hlo] += (dim & 1) ? -w : w;
        if (dim == 0) {
            rv[2 * (hmin - hlo)] += w;
        } else {
            int64_t s = (dim & 1) ? w : -w;
            rd[2 * (hmin - hlo) + 1] += s;
            rd[2 * (hmax - hlo)] -= s;
        }
    }
    int64_t nt = 0, nto = 0, ntc = 0, run = 0, rrun = 0, prev_e = 0, prev_r = 0;
    for (int64_t h = 0; h < R; ++h) {
        run += ect[h];
        if (run != prev_e) {
            if (T && nt < cap) { T[nt] = h + hlo; E[nt] = run; }
            ++nt;
            prev_e = run;
        }
        rrun += rd[2 * h];
        int64_t at = rv[2 * h] + rrun;
        rrun += rd[2 * h + 1];
        int64_t after = rrun;
        if (at != prev_r) {
            if (Tc && ntc < cap) { Tc[ntc] = h + hlo; Ec[ntc] = at; }
            ++ntc;
        }
        if (after != prev_r) {
            if (To && nto < cap) { To[nto] = h + hlo; Eo[nto] = after; }
            ++nto;
        }
        prev_r = after;
    }
    free(ect); free(rv); free(rd);
    if (nT) *nT = nt;
    if (nTo) *nTo = nto;
    if (nTc) *nTc = ntc;
    if ((T && nt > cap) || (To && nto > cap) || (Tc && ntc > cap)) return -2;
    return 0;
}

/* ---------------------------------------------------------------------------
 * Hybrid transform. HT(xi) = int kappa(t) Radon(xi, t) dt in the
 * paper's normalised height t: t(H) = (2H - L * csum) / (2L), with
 * csum = sum of xi_i over axes with M_i > 1 (E10, E11).
 *
 * Kernels kappa and a primitive kbar (E11): GAUSS: exp(-t^2/(2 s^2)),
 * s sqrt(pi/2) erf(t/(s sqrt2)); COS: cos(2 pi t / P), P/(2pi) sin(2 pi t/P);
 * SIN: sin t, -cos t; EXP: exp t, exp t (Appendix A);
 * ONE: 1, t.
 * ------------------------------------------------------------------------- */
static long double kappa(int kern, long double p, long double t)
{
    switch (kern) {
    case EO_GAUSS: return expl(-t * t / (2.0L * p * p));
    case EO_COS: return cosl(2.0L * 3.141592653589793238462643383279502884L * t / p);
    case EO_SIN: return sinl(t);
    case EO_EXP: return expl(t);
    default: return 1.0L;
    }
}

static long double kbar(int kern, long double p, long double t)
{
    const long double PI = 3.141592653589793238462643383279502884L;
    switch (kern) {
    case EO_GAUSS: return p * sqrtl(PI / 2.0L) * erfl(t / (p * sqrtl(2.0L)));
    case EO_COS: return p / (2.0L * PI) * sinl(2.0L * PI * t / p);
    case EO_SIN: return -cosl(t);
    case EO_EXP: return expl(t);
    default: return t;
    }
}

/* Neumaier-compensated accumulation in long double. */
typedef struct { long double s, c; } nsum;
static void nadd(nsum *a, long double x)
{
    long double t = a->s + x;
    if (fabsl(a->s) >= fabsl(x)) a->c += (a->s - t) + x; else a->c += (x - t) + a->s;
    a->s = t;
}

/* 8-node Gauss-Legendre nodes/weights on [-1,1]. */
static const long double GL_X[8] = {
    -0.9602898564975362316835608685694730L, -0.7966664774136267395915539364758304L,
    -0.5255324099163289858177390491892463L, -0.1834346424956498049394761423601840L,
     0.1834346424956498049394761423601840L,  0.5255324099163289858177390491892463L,
     0.7966664774136267395915539364758304L,  0.9602898564975362316835608685694730L};
static const long double GL_W[8] = {
    0.1012285362903762591525313543099622L, 0.2223810344533744705443559944262409L,
    0.3137066458778872873379622019866013L, 0.3626837833783619829651504492771810L,
    0.3626837833783619829651504492771810L, 0.3137066458778872873379622019866013L,
    0.2223810344533744705443559944262409L, 0.1012285362903762591525313543099622L};

static long double t_of(int64_t H, int64_t L, int64_t csum)
{
    return (long double)(2 * H - L * csum) / (long double)(2 * L);
}

/* Quadrature form (the definition): Radon is a step function constant on each
 * open interval (H, H+1) between lattice heights; integrate kappa over each
 * with 8-node Gauss-Legendre (ngl subdivisions) and weight by that constant.
 * Lattice-height points have measure zero. */
double eo_ht_quad(const int32_t *cells, int n, const int64_t *d, const int64_t *xs,
                  int64_t L, int64_t csum, int kern, double param, int nsub)
{
    int64_t ncell = 1, hlo = 0, hhi = 0;
    for (int i = 0; i < n; ++i) {
        ncell *= d[i];
        int64_t ext = xs[i] * ((d[i] - 1) / 2);
        if (ext < 0) hlo += ext; else hhi += ext;
    }
    int64_t R = hhi - hlo + 1;
    int64_t *rd = calloc((size_t)(2 * R + 2), sizeof(int64_t));
    if (!rd) return NAN;
    for (int64_t k = 0; k < ncell; ++k) {
        int64_t u[EO_MAXN], hmin, hmax;
        unrank(k, n, d, u);
        int dim = 0;
        for (int i = 0; i < n; ++i) dim += (int)(u[i] & 1);
        if (dim == 0) continue;
        cell_hrange(n, u, xs, &hmin, &hmax);
        int64_t w = cells[k];
        int64_t s = (dim & 1) ? w : -w;
        rd[2 * (hmin - hlo) + 1] += s;
        rd[2 * (hmax - hlo)] -= s;
    }
    nsum acc = {0, 0};
    int64_t run = 0;
    if (nsub < 1) nsub = 1;
    for (int64_t h = 0; h + 1 < R; ++h) {
        run += rd[2 * h] + rd[2 * h + 1]; /* value on (h, h+1) */
        if (run == 0) continue;
        long double a = t_of(h + hlo, L, csum), b = t_of(h + 1 + hlo, L, csum);
        long double wsub = (b - a) / nsub;
        nsum in = {0, 0};
        for (int s = 0; s < nsub; ++s) {
            long double a0 = a + s * wsub, half = wsub / 2, mid = a0 + half;
            for (int j = 0; j < 8; ++j) nadd(&in, GL_W[j] * half * kappa(kern, param, mid + half * GL_X[j]));
        }
        nadd(&acc, (long double)run * (in.s + in.c));
    }
    free(rd);
    return (double)(acc.s + acc.c);
}

/* Cell-primitive form (Lemma 1 with the (-1)^(dim-1) factor restored, E2):
 * HT = sum_{dim P >= 1} (-1)^(dim-1) phi(P) (kbar(t(max_P)) - kbar(t(min_P))). */
double eo_ht_cells(const int32_t *cells, int n, const int64_t *d, const int64_t *xs,
                   int64_t L, int64_t csum, int kern, double param)
{
    int64_t ncell = 1;
    for (int i = 0; i < n; ++i) ncell *= d[i];
    nsum acc = {0, 0};
    for (int64_t k = 0; k < ncell; ++k) {
        int64_t u[EO_MAXN], hmin, hmax;
        unrank(k, n, d, u);
        int dim = 0;
        for (int i = 0; i < n; ++i) dim += (int)(u[i] & 1);
        if (dim == 0 || cells[k] == 0) continue;
        cell_hrange(n, u, xs, &hmin, &hmax);
        long double s = (dim & 1) ? (long double)cells[k] : -(long double)cells[k];
        nadd(&acc, s * (kbar(kern, param, t_of(hmax, L, csum)) - kbar(kern, param, t_of(hmin, L, csum))));
    }
    return (double)(acc.s + acc.c);
}

/* ---------------------------------------------------------------------------
 * Real-valued directions (NEXT row f3; the paper's experimental setting,
 * P:140). Vertex p is embedded at x_i = p_i / (M_i - 1) - 0.5 (0 when
 * M_i = 1) and its height is the double
 *     h(p) = ((xi_0 x_0 + xi_1 x_1) + xi_2 x_2)
 * evaluated left to right in IEEE double, round to nearest, no fused
 * multiply-add (E22: ties are exact equalities of these identically
 * computed dots). A cell's heights are the min / max over its vertices.
 * The transforms are the same cell sums as eo_transforms (E2 / Lemma 4),
 * swept over the sorted distinct vertex heights c_0 < c_1 < ... (every
 * breakpoint is a vertex height): ECT at c_k counts the cells with
 * max_P <= c_k; Radon at c_k counts the vertices at c_k and the cells with
 * min_P < c_k < max_P, and on (c_k, c_{k+1}) the cells with min_P <= c_k and
 * max_P >= c_{k+1}. Canonical extraction as in eo_transforms.
 * ------------------------------------------------------------------------- */
static int cmp_double(const void *a, const void *b)
{
    double x = *(const double *)a, y = *(const double *)b;
    return x < y ? -1 : x > y ? 1 : 0;
}

static int64_t find_height(const double *c, int64_t nc, double h)
{
    int64_t lo = 0, hi = nc - 1;
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (c[mid] < h) lo = mid + 1; else hi = mid;
    }
    return lo; /* c[lo] == h: h is a vertex height */
}

static double vertex_height(int n, const int64_t *d, const int64_t *p, const double *xi)
{
    volatile double h = 0.0; /* volatile: keep the written order, no contraction */
    for (int i = 0; i < n; ++i) {
        const int64_t M = (d[i] + 1) / 2;
        volatile double x = M > 1 ? (double)p[i] / (double)(M - 1) : 0.0;
        if (M > 1) x = x - 0.5;
        volatile double t = xi[i] * x;
        h = (i == 0) ? t : h + t;
    }
    h = h + 0.0; /* -0.0 -> +0.0 */
    return h;
}

int eo_transforms_real(const int32_t *cells, int n, const int64_t *d, const double *xi, int64_t cap,
                       double *T, int64_t *E, int64_t *nT,
                       double *To, int64_t *Eo, int64_t *nTo,
                       double *Tc, int64_t *Ec, int64_t *nTc)
{
    if (n < 1 || n > EO_MAXN) return -1;
    int64_t ncell = 1, nv = 1, M[EO_MAXN];
    for (int i = 0; i < n; ++i) {
        ncell *= d[i];
        M[i] = (d[i] + 1) / 2;
        nv *= M[i];
    }
    double *vh = malloc(sizeof(double) * (size_t)nv), *c = malloc(sizeof(double) * (size_t)nv);
    if (!vh || !c) { free(vh); free(c); return -3; }
    for (int64_t k = 0; k < nv; ++k) {
        int64_t p[EO_MAXN];
        unrank(k, n, M, p);
        vh[k] = vertex_height(n, d, p, xi);
        c[k] = vh[k];
    }
    qsort(c, (size_t)nv, sizeof(double), cmp_double);
    int64_t nc = 0;
    for (int64_t k = 0; k < nv; ++k)
        if (nc == 0 || c[k] != c[nc - 1]) c[nc++] = c[k];
    int64_t *ect = calloc((size_t)nc + 1, sizeof(int64_t));
    int64_t *rv = calloc((size_t)nc + 1, sizeof(int64_t));
    int64_t *rd = calloc((size_t)(2 * nc + 2), sizeof(int64_t));
    if (!ect || !rv || !rd) { free(vh); free(c); free(ect); free(rv); free(rd); return -3; }
    for (int64_t k = 0; k < ncell; ++k) {
        int64_t u[EO_MAXN];
        unrank(k, n, d, u);
        int dim = 0;
        for (int i = 0; i < n; ++i) dim += (int)(u[i] & 1);
        /* the cell's vertices: u_i even -> u_i/2; odd -> (u_i-1)/2 and (u_i+1)/2 */
        double hmin = 0, hmax = 0;
        for (int mask = 0; mask < (1 << n); ++mask) {
            int64_t p[EO_MAXN];
            int dup = 0;
            for (int i = 0; i < n; ++i) {
                int bit = (mask >> i) & 1;
                if (u[i] % 2 == 0) { p[i] = u[i] / 2; if (bit) dup = 1; }
                else p[i] = (u[i] - 1) / 2 + bit;
            }
            if (dup) continue;
            double h = vh[rank_of(n, M, p)];
            if (mask == 0 || h < hmin) hmin = h;
            if (mask == 0 || h > hmax) hmax = h;
        }
        int64_t kmin = find_height(c, nc, hmin), kmax = find_height(c, nc, hmax);
        int64_t w = cells[k];
        ect[kmax] += (dim & 1) ? -w : w;
        if (dim == 0) {
            rv[kmin] += w;
        } else {
            /* (-1)^(dim-1) w on the open interval (hmin, hmax): on the points c_k with
               kmin < k < kmax and on the gaps (c_k, c_k+1) with kmin <= k < kmax */
            int64_t s = (dim & 1) ? w : -w;
            rd[2 * kmin + 1] += s;
            rd[2 * kmax] -= s;
        }
    }
    int64_t nt = 0, nto = 0, ntc = 0, run = 0, rrun = 0, prev_e = 0, prev_r = 0;
    for (int64_t k = 0; k < nc; ++k) {
        run += ect[k];
        if (run != prev_e) {
            if (T && nt < cap) { T[nt] = c[k]; E[nt] = run; }
            ++nt;
            prev_e = run;
        }
        rrun += rd[2 * k];
        int64_t at = rv[k] + rrun;
        rrun += rd[2 * k + 1];
        int64_t after = rrun;
        if (at != prev_r) {
            if (Tc && ntc < cap) { Tc[ntc] = c[k]; Ec[ntc] = at; }
            ++ntc;
        }
        if (after != prev_r) {
            if (To && nto < cap) { To[nto] = c[k]; Eo[nto] = after; }
            ++nto;
        }
        prev_r = after;
    }
    free(vh); free(c); free(ect); free(rv); free(rd);
    if (nT) *nT = nt;
    if (nTo) *nTo = nto;
    if (nTc) *nTc = ntc;
    if ((T && nt > cap) || (To && nto > cap) || (Tc && ntc > cap)) return -2;
    return 0;
}
