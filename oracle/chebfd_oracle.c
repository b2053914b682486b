/* CPU restatement of the ChebFD hot path -- TEST INFRASTRUCTURE ONLY.
 * See chebfd_oracle.h for the contract and the pinning strategy.
 * Citations are file:line relative to /root/reference/proj.
 * Built with -ffp-contract=off so no FMA contraction happens (the reference
 * is built for baseline x86-64, which has no FMA). */
#include "chebfd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.141592653589793238462643383279502884;

/* ------------------------------------------------------------------ RNG -- */
/* std::mt19937_64 (C++11 [rand.predef]): w=64 n=312 m=156 r=31,
 * a=0xB5026F5AA96619E9 u=29 d=0x5555555555555555 s=17 b=0x71D67FFFEDA60000
 * t=37 c=0xFFF7EEE000000000 l=43 f=6364136223846793005 */
void orc_rng_seed(orc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = 312;
    r->have_saved = 0;
    r->saved = 0.0;
}

static void mt_refill(orc_rng* r) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    const uint64_t a = 0xB5026F5AA96619E9ULL;
    for (int i = 0; i < 312; ++i) {
        uint64_t y = (r->mt[i] & upper) | (r->mt[(i + 1) % 312] & lower);
        r->mt[i] = r->mt[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? a : 0ULL);
    }
    r->mti = 0;
}

uint64_t orc_rng_next(orc_rng* r) {
    if (r->mti >= 312) mt_refill(r);
    uint64_t z = r->mt[r->mti++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

void orc_rng_discard(orc_rng* r, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) (void)orc_rng_next(r);
}

/* libstdc++ std::generate_canonical<double, 53>(mt19937_64): one draw,
 * (double)x / 2^64, clamped below 1 (bits/random.tcc). */
double orc_rng_canonical(orc_rng* r) {
    const double sum = (double)orc_rng_next(r);
    const double tmp = 18446744073709551616.0; /* 2^64 */
    double ret = sum / tmp;
    if (ret >= 1.0) ret = nextafter(1.0, 0.0);
    return ret;
}

/* libstdc++ std::normal_distribution<double>::operator() (Marsaglia polar,
 * caching the second variate), mean 0, stddev 1 (bits/random.tcc). */
double orc_rng_normal(orc_rng* r) {
    double ret;
    if (r->have_saved) {
        r->have_saved = 0;
        ret = r->saved;
    } else {
        double x, y, r2;
        do {
            x = 2.0 * orc_rng_canonical(r) - 1.0;
            y = 2.0 * orc_rng_canonical(r) - 1.0;
            r2 = x * x + y * y;
        } while (r2 > 1.0 || r2 == 0.0);
        const double mult = sqrt(-2.0 * log(r2) / r2);
        r->saved = x * mult;
        r->have_saved = 1;
        ret = y * mult;
    }
    return ret * 1.0 + 0.0;
}

/* BlockVector::randomize (block_vector.hpp:42-51).  For complex entries
 * `Complex(dist(gen), dist(gen))` -- GCC evaluates the two constructor
 * arguments right to left, so the IMAGINARY part is drawn first (pinned
 * against the compiled reference in tests/test_oracle.py). */
void orc_randomize(int kind, int64_t dim, int64_t width, uint64_t seed, void* out) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    double* o = (double*)out;
    const int64_t n = dim * width;
    if (kind == 0) {
        for (int64_t i = 0; i < n; ++i) o[i] = orc_rng_normal(&r);
    } else {
        for (int64_t i = 0; i < n; ++i) {
            const double im = orc_rng_normal(&r);
            const double re = orc_rng_normal(&r);
            o[2 * i] = re;
            o[2 * i + 1] = im;
        }
    }
}

/* box_draw (models.cpp:13-16) */
static double box_draw(orc_rng* r, double v) {
    const double u = (double)(orc_rng_next(r) >> 11) * 0x1p-53;
    return v * (u - 0.5);
}

/* ------------------------------------------- SparseMatrix::Builder ------ */
/* Builder (sparse_matrix.hpp:57-84): per-row std::map<col, S>, values
 * summed with `+=` starting from S{} in insertion order, rows emitted with
 * ascending columns.  Restated as a stable bucket sort of the triplets. */
typedef struct {
    int64_t row, col;
    double re, im;
} trip;

typedef struct {
    trip* t;
    int64_t n, cap;
} trip_list;

static void tl_add(trip_list* l, int64_t i, int64_t j, double re, double im) {
    if (l->n == l->cap) {
        l->cap = l->cap ? 2 * l->cap : 1024;
        l->t = (trip*)realloc(l->t, sizeof(trip) * (size_t)l->cap);
    }
    trip* p = &l->t[l->n++];
    p->row = i;
    p->col = j;
    p->re = re;
    p->im = im;
}

/* emits CSR; returns nnz.  When offs == NULL only counts. */
static int64_t tl_build(trip_list* l, int64_t dim, int kind, int64_t* offs, int64_t* cols,
                        double* vals) {
    int64_t* cnt = (int64_t*)calloc((size_t)dim + 1, sizeof(int64_t));
    for (int64_t k = 0; k < l->n; ++k) cnt[l->t[k].row + 1]++;
    for (int64_t i = 0; i < dim; ++i) cnt[i + 1] += cnt[i];
    trip* s = (trip*)malloc(sizeof(trip) * (size_t)(l->n ? l->n : 1));
    int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(dim + 1));
    memcpy(pos, cnt, sizeof(int64_t) * (size_t)(dim + 1));
    for (int64_t k = 0; k < l->n; ++k) s[pos[l->t[k].row]++] = l->t[k]; /* stable by row */
    int64_t nnz = 0;
    for (int64_t i = 0; i < dim; ++i) {
        const int64_t b = cnt[i], e = cnt[i + 1];
        /* stable insertion sort by column */
        for (int64_t k = b + 1; k < e; ++k) {
            trip x = s[k];
            int64_t m = k - 1;
            while (m >= b && s[m].col > x.col) {
                s[m + 1] = s[m];
                --m;
            }
            s[m + 1] = x;
        }
        if (offs) offs[i] = nnz;
        for (int64_t k = b; k < e;) {
            const int64_t c = s[k].col;
            double re = 0.0, im = 0.0; /* S{} then += in insertion order */
            while (k < e && s[k].col == c) {
                re += s[k].re;
                im += s[k].im;
                ++k;
            }
            if (cols) {
                cols[nnz] = c;
                if (kind == 0) {
                    vals[nnz] = re;
                } else {
                    vals[2 * nnz] = re;
                    vals[2 * nnz + 1] = im;
                }
            }
            ++nnz;
        }
    }
    if (offs) offs[dim] = nnz;
    free(cnt);
    free(s);
    free(pos);
    return nnz;
}

/* ------------------------------------------------------------ models ---- */
/* graphene (models.cpp:142-178) */
int orc_graphene(int64_t lx, int64_t ly, double t, double disorder, int boundary, uint64_t seed,
                 int64_t* dim_out, int64_t* nnz_out, int64_t* offs, int64_t* cols,
                 double* vals) {
    if (lx < 1 || ly < 1 || disorder < 0.0) return 1; /* LatticeSpec::validate :7-13 */
    const int64_t dim = 2 * lx * ly;
    const int periodic = boundary != 2;
    double* vn = (double*)malloc(sizeof(double) * (size_t)dim);
    orc_rng r;
    orc_rng_seed(&r, seed);
    for (int64_t n = 0; n < dim; ++n) vn[n] = box_draw(&r, disorder);
    trip_list l = {0, 0, 0};
    for (int64_t y = 0; y < ly; ++y)
        for (int64_t x = 0; x < lx; ++x) {
            const int64_t a = 2 * (x + lx * y);
            tl_add(&l, a, a, vn[a], 0.0);
            tl_add(&l, a + 1, a + 1, vn[a + 1], 0.0);
            /* bonds to B in the same cell, the cell at x-1 and the cell at y-1 */
            const int64_t bx[3] = {x, x - 1, x};
            const int64_t by[3] = {y, y, y - 1};
            const int wrap[3] = {0, x == 0, y == 0};
            for (int k = 0; k < 3; ++k) {
                if (wrap[k] && !periodic) continue;
                const int64_t bb = 2 * ((bx[k] + lx) % lx + lx * ((by[k] + ly) % ly)) + 1;
                tl_add(&l, a, bb, -t, 0.0);
                tl_add(&l, bb, a, -t, 0.0);
            }
        }
    free(vn);
    *dim_out = dim;
    *nnz_out = tl_build(&l, dim, 0, offs, cols, vals);
    free(l.t);
    return 0;
}

/* complex helpers with GCC's inline expansion order for _Complex double */
static void cmul(double ar, double ai, double br, double bi, double* cr, double* ci) {
    *cr = ar * br - ai * bi;
    *ci = ar * bi + ai * br;
}

/* gamma_matrices (models.cpp:45-57): G0 = tz x s0, G1 = tx x s0,
 * G2 = ty x sx, G3 = ty x sy, G4 = ty x sz.  kron (:25-32). */
static void gamma_set(double g[5][4][4][2]) {
    double s0[2][2][2] = {{{1, 0}, {0, 0}}, {{0, 0}, {1, 0}}};
    double sx[2][2][2] = {{{0, 0}, {1, 0}}, {{1, 0}, {0, 0}}};
    double sy[2][2][2] = {{{0, 0}, {0, -1}}, {{0, 1}, {0, 0}}};
    double sz[2][2][2] = {{{1, 0}, {0, 0}}, {{0, 0}, {-1, 0}}};
    double (*tau[5])[2][2] = {sz, sx, sy, sy, sy};
    double (*sig[5])[2][2] = {s0, s0, sx, sy, sz};
    for (int q = 0; q < 5; ++q)
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b)
                for (int c = 0; c < 2; ++c)
                    for (int d = 0; d < 2; ++d)
                        cmul(tau[q][a][b][0], tau[q][a][b][1], sig[q][c][d][0], sig[q][c][d][1],
                             &g[q][2 * a + c][2 * b + d][0], &g[q][2 * a + c][2 * b + d][1]);
}

/* topological_insulator (models.cpp:80-140) */
int orc_topological_insulator(int64_t lx, int64_t ly, int64_t lz, double t, double disorder,
                              int boundary, uint64_t seed, int64_t* dim_out, int64_t* nnz_out,
                              int64_t* offs, int64_t* cols, double* vals) {
    if (lx < 1 || ly < 1 || lz < 1 || disorder < 0.0) return 1;
    const int64_t ns = lx * ly * lz;
    const int64_t dim = 4 * ns;
    double g[5][4][4][2];
    gamma_set(g);
    /* hop[j] = -t (G1 - i G^{j+1}) / 2  (:87-92) */
    double hop[3][4][4][2];
    for (int j = 0; j < 3; ++j)
        for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) {
                double ir, ii; /* I * G[j+2] */
                cmul(0.0, 1.0, g[j + 2][r][c][0], g[j + 2][r][c][1], &ir, &ii);
                const double dr = g[1][r][c][0] - ir, di = g[1][r][c][1] - ii;
                const double s = -t * 0.5;
                hop[j][r][c][0] = s * dr;
                hop[j][r][c][1] = s * di;
            }
    double* vn = (double*)malloc(sizeof(double) * (size_t)ns);
    orc_rng rng;
    orc_rng_seed(&rng, seed);
    for (int64_t n = 0; n < ns; ++n) vn[n] = box_draw(&rng, disorder);
    const int per_xy = boundary != 2, per_z = boundary == 1;
    const int periodic[3] = {per_xy, per_xy, per_z};
    const int64_t len[3] = {lx, ly, lz};
    trip_list l = {0, 0, 0};
    for (int64_t z = 0; z < lz; ++z)
        for (int64_t y = 0; y < ly; ++y)
            for (int64_t x = 0; x < lx; ++x) {
                const int64_t n = x + lx * (y + ly * z);
                for (int r = 0; r < 4; ++r) {
                    tl_add(&l, 4 * n + r, 4 * n + r, vn[n] * g[0][r][r][0], vn[n] * g[0][r][r][1]);
                    for (int c = 0; c < 4; ++c) {
                        const double vr = 2.0 * g[1][r][c][0], vi = 2.0 * g[1][r][c][1];
                        if (r != c && !(vr == 0.0 && vi == 0.0)) tl_add(&l, 4 * n + r, 4 * n + c, vr, vi);
                    }
                }
                const int64_t pos[3] = {x, y, z};
                for (int j = 0; j < 3; ++j) {
                    int64_t pj = pos[j] + 1;
                    if (pj == len[j]) {
                        if (!periodic[j] || len[j] == 1) continue;
                        pj = 0;
                    }
                    int64_t q[3] = {x, y, z};
                    q[j] = pj;
                    const int64_t m = q[0] + lx * (q[1] + ly * q[2]);
                    for (int r = 0; r < 4; ++r)
                        for (int c = 0; c < 4; ++c) {
                            const double vr = hop[j][r][c][0], vi = hop[j][r][c][1];
                            if (vr == 0.0 && vi == 0.0) continue;
                            tl_add(&l, 4 * m + r, 4 * n + c, vr, vi);
                            tl_add(&l, 4 * n + c, 4 * m + r, vr, -vi);
                        }
                }
            }
    free(vn);
    *dim_out = dim;
    *nnz_out = tl_build(&l, dim, 1, offs, cols, vals);
    free(l.t);
    return 0;
}

/* ------------------------------------------------- filter coefficients -- */
/* window_coeffs (filter.cpp:43-56) */
int orc_window_coeffs(double tlo, double thi, double blo, double bhi, int degree, double* c) {
    if (!(tlo < thi) || !(blo < bhi) || !(blo <= tlo && thi <= bhi)) return 1;
    if (degree < 1) return 1;
    const double alpha = 2.0 / (bhi - blo);
    const double beta = (blo + bhi) / (blo - bhi);
    double xl = alpha * tlo + beta, xh = alpha * thi + beta;
    xl = xl < -1.0 ? -1.0 : (xl > 1.0 ? 1.0 : xl);
    xh = xh < -1.0 ? -1.0 : (xh > 1.0 ? 1.0 : xh);
    const double a_lo = acos(xl), a_hi = acos(xh);
    c[0] = (a_lo - a_hi) / kPi;
    for (int n = 1; n <= degree; ++n) c[n] = 2.0 / (kPi * n) * (sin(n * a_lo) - sin(n * a_hi));
    return 0;
}

/* kernel_coeffs (filter.cpp:58-84) */
int orc_kernel_coeffs(int kind, int mu, int degree, double* g) {
    if (degree < 1) return 1;
    const int np = degree;
    for (int n = 0; n <= np; ++n) g[n] = 1.0;
    switch (kind) {
        case 0: break;
        case 1:
            for (int n = 0; n <= np; ++n) g[n] = (double)(np - n + 1) / (np + 1);
            break;
        case 2: {
            const double cot = cos(kPi / np) / sin(kPi / np);
            for (int n = 0; n <= np; ++n)
                g[n] = ((np - n) * cos(kPi * n / np) + sin(kPi * n / np) * cot) / np;
            break;
        }
        case 3:
            if (mu < 1) return 1;
            for (int n = 1; n <= np; ++n) {
                const double x = kPi * n / (np + 1);
                g[n] = pow(sin(x) / x, (double)mu);
            }
            break;
        default: return 1;
    }
    return 0;
}

/* make_filter (filter.cpp:86-99) */
int orc_make_filter(double tlo, double thi, double blo, double bhi, int degree, int kind, int mu,
                    double* combined, double* alpha, double* beta) {
    *alpha = 2.0 / (bhi - blo);
    *beta = (blo + bhi) / (blo - bhi);
    double* c = (double*)malloc(sizeof(double) * (size_t)(degree + 1));
    double* g = (double*)malloc(sizeof(double) * (size_t)(degree + 1));
    int rc = orc_window_coeffs(tlo, thi, blo, bhi, degree, c);
    if (!rc) rc = orc_kernel_coeffs(kind, mu, degree, g);
    if (!rc)
        for (int n = 0; n <= degree; ++n) combined[n] = g[n] * c[n];
    free(c);
    free(g);
    return rc;
}

/* eval_scalar (filter.cpp:101-114), bounds check left to the caller */
double orc_eval_scalar(const double* cmb, int degree, double alpha, double beta, double x) {
    const double t = alpha * x + beta;
    double tm2 = 1.0, tm1 = t;
    double acc = cmb[0] + cmb[1] * t;
    for (int n = 2; n <= degree; ++n) {
        const double tn = 2.0 * t * tm1 - tm2;
        acc += cmb[n] * tn;
        tm2 = tm1;
        tm1 = tn;
    }
    return acc;
}

/* -------------------------------------------------------------- kernels -- */
/* spmmvm (kernels.hpp:45-69): Y = (alpha A + beta I) X, Y zero-filled */
int orc_spmmvm(const orc_csr* a, const double* x, int64_t nb, double alpha, double beta,
               double* y) {
    const int cx = a->kind == 1;
    const int64_t w = cx ? 2 * nb : nb;
    memset(y, 0, sizeof(double) * (size_t)(a->dim * w));
    for (int64_t i = 0; i < a->dim; ++i) {
        double* yi = y + i * w;
        for (int64_t p = a->offs[i]; p < a->offs[i + 1]; ++p) {
            const double* xj = x + a->cols[p] * w;
            if (!cx) {
                const double av = a->vals[p] * alpha;
                for (int64_t k = 0; k < nb; ++k) yi[k] += av * xj[k];
            } else {
                const double ar = a->vals[2 * p] * alpha, ai = a->vals[2 * p + 1] * alpha;
                for (int64_t k = 0; k < nb; ++k) {
                    double pr, pi;
                    cmul(ar, ai, xj[2 * k], xj[2 * k + 1], &pr, &pi);
                    yi[2 * k] += pr;
                    yi[2 * k + 1] += pi;
                }
            }
        }
        if (beta != 0.0) {
            const double* xi = x + i * w;
            for (int64_t k = 0; k < w; ++k) yi[k] += beta * xi[k];
        }
    }
    return 0;
}

/* Kahan (kernels.hpp:12-23), componentwise for complex */
typedef struct {
    double s, c;
} kahan;
static void kahan_add(kahan* k, double v) {
    const double y = v - k->c;
    const double t = k->s + y;
    k->c = (t - k->s) - y;
    k->s = t;
}

/* spmmvm_fused (kernels.hpp:71-118) with one row chunk */
int orc_spmmvm_fused(const orc_csr* a, const double* u, double* w, double* x, int64_t nb,
                     double alpha, double beta, double coeff, double* dots) {
    if (u == w || u == x || w == x) return 1; /* aliasing guard :80-81 */
    const int cx = a->kind == 1;
    const int64_t wd = cx ? 2 * nb : nb;
    double* tmp = (double*)malloc(sizeof(double) * (size_t)wd);
    kahan* acc = dots ? (kahan*)calloc((size_t)wd, sizeof(kahan)) : NULL;
    for (int64_t i = 0; i < a->dim; ++i) {
        for (int64_t k = 0; k < wd; ++k) tmp[k] = 0.0;
        for (int64_t p = a->offs[i]; p < a->offs[i + 1]; ++p) {
            const double* uj = u + a->cols[p] * wd;
            if (!cx) {
                const double av = a->vals[p] * (2.0 * alpha);
                for (int64_t k = 0; k < nb; ++k) tmp[k] += av * uj[k];
            } else {
                const double ar = a->vals[2 * p] * (2.0 * alpha);
                const double ai = a->vals[2 * p + 1] * (2.0 * alpha);
                for (int64_t k = 0; k < nb; ++k) {
                    double pr, pi;
                    cmul(ar, ai, uj[2 * k], uj[2 * k + 1], &pr, &pi);
                    tmp[2 * k] += pr;
                    tmp[2 * k + 1] += pi;
                }
            }
        }
        double* wi = w + i * wd;
        double* xi = x + i * wd;
        const double* ui = u + i * wd;
        for (int64_t k = 0; k < nb; ++k) {
            if (!cx) {
                const double wn = tmp[k] + (2.0 * beta) * ui[k] - wi[k];
                wi[k] = wn;
                if (acc) kahan_add(&acc[k], xi[k] * wn);
                xi[k] += coeff * wn;
            } else {
                const double wr = tmp[2 * k] + (2.0 * beta) * ui[2 * k] - wi[2 * k];
                const double wim = tmp[2 * k + 1] + (2.0 * beta) * ui[2 * k + 1] - wi[2 * k + 1];
                wi[2 * k] = wr;
                wi[2 * k + 1] = wim;
                if (acc) {
                    double pr, pi;
                    cmul(xi[2 * k], -xi[2 * k + 1], wr, wim, &pr, &pi);
                    /* Kahan<Complex>::add: complex ops are componentwise */
                    kahan_add(&acc[2 * k], pr);
                    kahan_add(&acc[2 * k + 1], pi);
                }
                xi[2 * k] += coeff * wr;
                xi[2 * k + 1] += coeff * wim;
            }
        }
    }
    if (dots) {
        /* chunk-ordered Kahan over one chunk (:110-117) */
        for (int64_t k = 0; k < wd; ++k) {
            kahan tot = {0.0, 0.0};
            kahan_add(&tot, acc[k].s);
            dots[k] = tot.s;
        }
    }
    free(tmp);
    free(acc);
    return 0;
}

/* recurrence_step (kernels.hpp:120-145) */
int orc_recurrence_step(const orc_csr* a, const double* u, double* w, int64_t nb, double alpha,
                        double beta) {
    if (u == w) return 1;
    const int cx = a->kind == 1;
    const int64_t wd = cx ? 2 * nb : nb;
    double* tmp = (double*)malloc(sizeof(double) * (size_t)wd);
    for (int64_t i = 0; i < a->dim; ++i) {
        for (int64_t k = 0; k < wd; ++k) tmp[k] = 0.0;
        for (int64_t p = a->offs[i]; p < a->offs[i + 1]; ++p) {
            const double* uj = u + a->cols[p] * wd;
            if (!cx) {
                const double av = a->vals[p] * (2.0 * alpha);
                for (int64_t k = 0; k < nb; ++k) tmp[k] += av * uj[k];
            } else {
                const double ar = a->vals[2 * p] * (2.0 * alpha);
                const double ai = a->vals[2 * p + 1] * (2.0 * alpha);
                for (int64_t k = 0; k < nb; ++k) {
                    double pr, pi;
                    cmul(ar, ai, uj[2 * k], uj[2 * k + 1], &pr, &pi);
                    tmp[2 * k] += pr;
                    tmp[2 * k + 1] += pi;
                }
            }
        }
        double* wi = w + i * wd;
        const double* ui = u + i * wd;
        for (int64_t k = 0; k < wd; ++k) wi[k] = tmp[k] + (2.0 * beta) * ui[k] - wi[k];
    }
    free(tmp);
    return 0;
}

/* block_axpy_scal (kernels.hpp:147-162): X = c0 X + c1 U + c2 W */
void orc_block_axpy_scal(int kind, int64_t dim, int64_t nb, double* x, const double* u,
                         const double* w, double c0, double c1, double c2) {
    const int64_t n = dim * nb * (kind == 1 ? 2 : 1);
    for (int64_t i = 0; i < n; ++i) x[i] = c0 * x[i] + c1 * u[i] + c2 * w[i];
}

/* column_dots (kernels.hpp:194-213), one chunk: d_k = sum conj(x) y */
void orc_column_dots(int kind, int64_t dim, int64_t nb, const double* x, const double* y,
                     double* d) {
    if (kind == 0) {
        for (int64_t k = 0; k < nb; ++k) d[k] = 0.0;
        double* acc = (double*)calloc((size_t)nb, sizeof(double));
        for (int64_t i = 0; i < dim; ++i)
            for (int64_t k = 0; k < nb; ++k) acc[k] += x[i * nb + k] * y[i * nb + k];
        for (int64_t k = 0; k < nb; ++k) d[k] += acc[k];
        free(acc);
    } else {
        double* acc = (double*)calloc((size_t)(2 * nb), sizeof(double));
        for (int64_t i = 0; i < dim; ++i)
            for (int64_t k = 0; k < nb; ++k) {
                double pr, pi;
                const double* xi = x + 2 * (i * nb + k);
                const double* yi = y + 2 * (i * nb + k);
                cmul(xi[0], -xi[1], yi[0], yi[1], &pr, &pi);
                acc[2 * k] += pr;
                acc[2 * k + 1] += pi;
            }
        for (int64_t k = 0; k < 2 * nb; ++k) d[k] = 0.0 + acc[k];
        free(acc);
    }
}

/* gram (kernels.hpp:164-192), one chunk, Kahan */
void orc_gram(int kind, int64_t dim, const double* x, int64_t nx, const double* y, int64_t ny,
              double* g) {
    const int cx = kind == 1;
    const int64_t m = nx * ny * (cx ? 2 : 1);
    kahan* acc = (kahan*)calloc((size_t)m, sizeof(kahan));
    for (int64_t i = 0; i < dim; ++i)
        for (int64_t k = 0; k < nx; ++k)
            for (int64_t l = 0; l < ny; ++l) {
                if (!cx) {
                    kahan_add(&acc[k * ny + l], x[i * nx + k] * y[i * ny + l]);
                } else {
                    double pr, pi;
                    const double* xk = x + 2 * (i * nx + k);
                    const double* yl = y + 2 * (i * ny + l);
                    cmul(xk[0], -xk[1], yl[0], yl[1], &pr, &pi);
                    kahan_add(&acc[2 * (k * ny + l)], pr);
                    kahan_add(&acc[2 * (k * ny + l) + 1], pi);
                }
            }
    for (int64_t q = 0; q < m; ++q) {
        kahan tot = {0.0, 0.0};
        kahan_add(&tot, acc[q].s);
        g[q] = tot.s;
    }
    free(acc);
}

/* block_mult_small (kernels.hpp:215-232): Y = X B */
void orc_block_mult_small(int kind, int64_t dim, int64_t nb, const double* x, const double* b,
                          int64_t bc, double* y) {
    const int cx = kind == 1;
    memset(y, 0, sizeof(double) * (size_t)(dim * bc * (cx ? 2 : 1)));
    for (int64_t i = 0; i < dim; ++i)
        for (int64_t k = 0; k < nb; ++k) {
            if (!cx) {
                const double xk = x[i * nb + k];
                for (int64_t j = 0; j < bc; ++j) y[i * bc + j] += xk * b[k * bc + j];
            } else {
                const double xr = x[2 * (i * nb + k)], xi = x[2 * (i * nb + k) + 1];
                for (int64_t j = 0; j < bc; ++j) {
                    double pr, pi;
                    cmul(xr, xi, b[2 * (k * bc + j)], b[2 * (k * bc + j) + 1], &pr, &pi);
                    y[2 * (i * bc + j)] += pr;
                    y[2 * (i * bc + j) + 1] += pi;
                }
            }
        }
}

/* column_norms (kernels.hpp:234-240) */
void orc_column_norms(int kind, int64_t dim, int64_t nb, const double* x, double* out) {
    double* d = (double*)malloc(sizeof(double) * (size_t)(nb * (kind == 1 ? 2 : 1)));
    orc_column_dots(kind, dim, nb, x, x, d);
    for (int64_t k = 0; k < nb; ++k) out[k] = sqrt(kind == 1 ? d[2 * k] : d[k]);
    free(d);
}

/* ------------------------------------------------------- apply_filter -- */
/* apply_filter (filter.hpp:73-116) */
int orc_apply_filter(const orc_csr* a, double* x, int64_t nb, const double* cmb, int degree,
                     double alpha, double beta, double* moments) {
    if (degree < 2) return 1;
    const int cx = a->kind == 1;
    const int64_t n = a->dim * nb * (cx ? 2 : 1);
    double* x0 = NULL;
    double* d = (double*)malloc(sizeof(double) * (size_t)(2 * nb));
    if (moments) {
        x0 = (double*)malloc(sizeof(double) * (size_t)n);
        memcpy(x0, x, sizeof(double) * (size_t)n);
        orc_column_dots(a->kind, a->dim, nb, x0, x0, d);
        for (int64_t k = 0; k < nb; ++k) moments[k] = cx ? d[2 * k] : d[k];
    }
    double* u = (double*)malloc(sizeof(double) * (size_t)n);
    double* w = (double*)malloc(sizeof(double) * (size_t)n);
    orc_spmmvm(a, x, nb, alpha, beta, u);
    orc_spmmvm(a, u, nb, 2.0 * alpha, 2.0 * beta, w);
    orc_block_axpy_scal(a->kind, a->dim, nb, w, x, x, 1.0, -1.0, 0.0);
    if (moments) {
        orc_column_dots(a->kind, a->dim, nb, x0, u, d);
        for (int64_t k = 0; k < nb; ++k) moments[nb + k] = cx ? d[2 * k] : d[k];
        orc_column_dots(a->kind, a->dim, nb, x0, w, d);
        for (int64_t k = 0; k < nb; ++k) moments[2 * nb + k] = cx ? d[2 * k] : d[k];
    }
    orc_block_axpy_scal(a->kind, a->dim, nb, x, u, w, cmb[0], cmb[1], cmb[2]);
    double* pu = u;
    double* pw = w;
    for (int k = 3; k <= degree; ++k) {
        double* t = pu;
        pu = pw;
        pw = t;
        orc_spmmvm_fused(a, pu, pw, x, nb, alpha, beta, cmb[k], NULL);
        if (moments) {
            orc_column_dots(a->kind, a->dim, nb, x0, pw, d);
            for (int64_t q = 0; q < nb; ++q) moments[k * nb + q] = cx ? d[2 * q] : d[q];
        }
    }
    free(u);
    free(w);
    free(x0);
    free(d);
    return 0;
}

/* bench.cpp:28-34 */
double orc_per_row_flops(double n_nzr, int f_a, int f_m) {
    return n_nzr * (f_a + f_m) + ceil(9.0 * f_a / 2.0) + ceil(11.0 * f_m / 2.0);
}
double orc_per_row_bytes(double n_nzr, int s_d, int s_i, int n_b) {
    return n_nzr / n_b * (s_d + s_i) + 5.0 * s_d;
}
