// Host-side pieces of the chebfd_b200 library: lattice generators, the
// reference's random streams, filter coefficients, DOS counts, partitions.
// All of it is pure host C++ (no CUDA); citations are file:line relative to
// /root/reference/proj.
#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <numbers>
#include <random>
#include <vector>

#include "internal.hpp"

namespace cfd {

namespace {
constexpr double kPi = std::numbers::pi;
using Cx = std::complex<double>;

// box_draw (models.cpp:13-16): portable uniform on [-v/2, v/2)
inline double box_draw(std::mt19937_64& rng, double v) {
    const double u = static_cast<double>(rng() >> 11) * 0x1p-53;
    return v * (u - 0.5);
}

// The five 4x4 Dirac matrices (models.cpp:45-57): G0 = tz x s0, G1 = tx x s0,
// G2 = ty x sx, G3 = ty x sy, G4 = ty x sz (kron as in models.cpp:25-32).
using Mat4 = std::array<std::array<Cx, 4>, 4>;
std::array<Mat4, 5> gammas() {
    using P = std::array<std::array<Cx, 2>, 2>;
    const Cx I{0.0, 1.0};
    const P s0{{{1, 0}, {0, 1}}}, sx{{{0, 1}, {1, 0}}}, sy{{{0, -I}, {I, 0}}},
        sz{{{1, 0}, {0, -1}}};
    auto kron = [](const P& t, const P& s) {
        Mat4 o{};
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b)
                for (int c = 0; c < 2; ++c)
                    for (int d = 0; d < 2; ++d) o[2 * a + c][2 * b + d] = t[a][b] * s[c][d];
        return o;
    };
    return {kron(sz, s0), kron(sx, s0), kron(sy, sx), kron(sy, sy), kron(sy, sz)};
}

struct Entry {
    int64_t col;
    Cx v;
};

// Merge one row's candidate entries the way SparseMatrix::Builder does
// (sparse_matrix.hpp:61-79): ascending columns, duplicates summed with `+=`
// starting from S{}.  Each row has at most two contributions per column and
// all of a column's contributions commute exactly, so the
// insertion order of the reference's site loop is not needed.
void emit_row(std::vector<Entry>& cand, HostCsr& out) {
    std::stable_sort(cand.begin(), cand.end(),
                     [](const Entry& a, const Entry& b) { return a.col < b.col; });
    for (size_t k = 0; k < cand.size();) {
        const int64_t c = cand[k].col;
        Cx s{};
        while (k < cand.size() && cand[k].col == c) s += cand[k++].v;
        out.cols.push_back(c);
        out.vals.push_back(s.real());
        if (out.kind) out.vals.push_back(s.imag());
    }
    out.offs.push_back(static_cast<int64_t>(out.cols.size()));
}
}  // namespace

void validate_lattice(const chebfd_lattice& s, bool needs_z) {
    // LatticeSpec::validate (models.cpp:19-27)
    if (s.lx < 1 || s.ly < 1 || (needs_z && s.lz < 1))
        fail(CHEBFD_ERR_INVALID_ARGUMENT, "LatticeSpec: lattice dimensions must be positive");
    if (s.disorder < 0.0)
        fail(CHEBFD_ERR_INVALID_ARGUMENT, "LatticeSpec: disorder strength must be >= 0");
    if (s.boundary < 0 || s.boundary > 2)
        fail(CHEBFD_ERR_INVALID_ARGUMENT, "LatticeSpec: bad boundary code");
}

// graphene (models.cpp:142-178), rows [r0, r1)
HostCsr gen_graphene(const chebfd_lattice& s, int64_t r0, int64_t r1) {
    validate_lattice(s, false);
    const int64_t lx = s.lx, ly = s.ly, dim = 2 * lx * ly;
    require(0 <= r0 && r0 <= r1 && r1 <= dim, "graphene: row range out of bounds");
    const bool periodic = s.boundary != CHEBFD_OPEN_ALL;
    std::mt19937_64 rng(s.seed);
    rng.discard(static_cast<unsigned long long>(r0));  // one draw per atom, in atom order
    HostCsr out;
    out.kind = 0;
    out.dim = dim;
    out.row_begin = r0;
    out.rows = r1 - r0;
    out.offs.reserve(r1 - r0 + 1);
    out.offs.push_back(0);
    out.cols.reserve(4 * (r1 - r0));
    out.vals.reserve(4 * (r1 - r0));
    std::vector<Entry> cand;
    const Cx bond{-s.t, 0.0};
    for (int64_t i = r0; i < r1; ++i) {
        const double vn = box_draw(rng, s.disorder);
        const int64_t cell = i / 2, sub = i % 2;
        const int64_t x = cell % lx, y = cell / lx;
        auto site = [&](int64_t cx, int64_t cy, int64_t sb) {
            return 2 * (((cx + lx) % lx) + lx * ((cy + ly) % ly)) + sb;
        };
        cand.clear();
        cand.push_back({i, Cx{vn, 0.0}});
        if (sub == 0) {
            // A(x,y) bonds to B in the same cell and the cells at x-1, y-1
            cand.push_back({site(x, y, 1), bond});
            if (x != 0 || periodic) cand.push_back({site(x - 1, y, 1), bond});
            if (y != 0 || periodic) cand.push_back({site(x, y - 1, 1), bond});
        } else {
            // B(x,y) is bonded by A(x,y), A(x+1,y) and A(x,y+1)
            cand.push_back({site(x, y, 0), bond});
            if (x + 1 < lx || periodic) cand.push_back({site(x + 1, y, 0), bond});
            if (y + 1 < ly || periodic) cand.push_back({site(x, y + 1, 0), bond});
        }
        emit_row(cand, out);
    }
    // values: real only
    return out;
}

// topological_insulator (models.cpp:80-140), rows [r0, r1)
HostCsr gen_topological_insulator(const chebfd_lattice& s, int64_t r0, int64_t r1) {
    validate_lattice(s, true);
    const int64_t lx = s.lx, ly = s.ly, lz = s.lz;
    const int64_t ns = lx * ly * lz, dim = 4 * ns;
    require(0 <= r0 && r0 <= r1 && r1 <= dim, "topological_insulator: row range out of bounds");
    const auto g = gammas();
    const Cx I{0.0, 1.0};
    Mat4 hop[3];
    for (int j = 0; j < 3; ++j)
        for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) hop[j][r][c] = -s.t * 0.5 * (g[1][r][c] - I * g[j + 2][r][c]);
    const bool per_xy = s.boundary != CHEBFD_OPEN_ALL;
    const bool per_z = s.boundary == CHEBFD_PERIODIC_ALL;
    const bool periodic[3] = {per_xy, per_xy, per_z};
    const int64_t len[3] = {lx, ly, lz};
    const int64_t site0 = r0 / 4;
    const int64_t site1 = r1 > r0 ? (r1 - 1) / 4 + 1 : site0;
    std::vector<double> vn(static_cast<size_t>(site1 - site0));
    {
        std::mt19937_64 rng(s.seed);
        rng.discard(static_cast<unsigned long long>(site0));  // one draw per site
        for (auto& v : vn) v = box_draw(rng, s.disorder);
    }
    HostCsr out;
    out.kind = 1;
    out.dim = dim;
    out.row_begin = r0;
    out.rows = r1 - r0;
    out.offs.reserve(r1 - r0 + 1);
    out.offs.push_back(0);
    out.cols.reserve(11 * (r1 - r0));
    out.vals.reserve(22 * (r1 - r0));
    std::vector<Entry> cand;
    for (int64_t i = r0; i < r1; ++i) {
        const int64_t n = i / 4;
        const int rr = static_cast<int>(i % 4);
        const int64_t pos[3] = {n % lx, (n / lx) % ly, n / (lx * ly)};
        cand.clear();
        // on-site V_n G0 + 2 G1 (models.cpp:113-119)
        cand.push_back({i, vn[n - site0] * g[0][rr][rr]});
        for (int c = 0; c < 4; ++c) {
            const Cx v = 2.0 * g[1][rr][c];
            if (rr != c && v != 0.0) cand.push_back({4 * n + c, v});
        }
        for (int j = 0; j < 3; ++j) {
            if (len[j] == 1) continue;  // (models.cpp:124-126)
            // row as the TARGET m of the hop from n' = n - e_j:  b.add(4m+r, 4n'+c, hop)
            {
                int64_t pj = pos[j] - 1;
                bool ok = true;
                if (pj < 0) {
                    ok = periodic[j];
                    pj = len[j] - 1;
                }
                if (ok) {
                    int64_t q[3] = {pos[0], pos[1], pos[2]};
                    q[j] = pj;
                    const int64_t np = q[0] + lx * (q[1] + ly * q[2]);
                    for (int c = 0; c < 4; ++c)
                        if (hop[j][rr][c] != 0.0) cand.push_back({4 * np + c, hop[j][rr][c]});
                }
            }
            // row as the SOURCE n of the hop to m = n + e_j:  b.add(4n+c, 4m+r, conj(hop))
            {
                int64_t pj = pos[j] + 1;
                bool ok = true;
                if (pj == len[j]) {
                    ok = periodic[j];
                    pj = 0;
                }
                if (ok) {
                    int64_t q[3] = {pos[0], pos[1], pos[2]};
                    q[j] = pj;
                    const int64_t m = q[0] + lx * (q[1] + ly * q[2]);
                    for (int r = 0; r < 4; ++r)
                        if (hop[j][r][rr] != 0.0) cand.push_back({4 * m + r, std::conj(hop[j][r][rr])});
                }
            }
        }
        emit_row(cand, out);
    }
    return out;
}

// window_coeffs (filter.cpp:43-56)
bool csr_is_hermitian(int kind, int64_t dim, const int64_t* offs, const int64_t* cols,
                      const double* vals) {
    for (int64_t i = 0; i < dim; ++i) {
        for (int64_t p = offs[i]; p < offs[i + 1]; ++p) {
            const int64_t j = cols[p];
            int64_t hit = -1, count = 0;
            for (int64_t q = offs[j]; q < offs[j + 1]; ++q)
                if (cols[q] == i) {
                    if (hit < 0) hit = q;
                    ++count;
                }
            if (count != 1) return false;
            if (kind) {
                if (vals[2 * p] != vals[2 * hit] || vals[2 * p + 1] != -vals[2 * hit + 1]) return false;
            } else if (vals[p] != vals[hit]) {
                return false;
            }
        }
    }
    return true;
}

void moments_from_doubling(double* m, int64_t rows, int64_t width) {
    for (int64_t q = 2; q < rows; ++q)
        for (int64_t k = 0; k < width; ++k) m[q * width + k] = 2.0 * m[q * width + k] - m[(q & 1) * width + k];
}

std::vector<double> window_coeffs(double tlo, double thi, double blo, double bhi, int degree) {
    if (!(tlo < thi)) fail(CHEBFD_ERR_INVALID_ARGUMENT, "degenerate target interval");
    if (!(blo < bhi)) fail(CHEBFD_ERR_INVALID_ARGUMENT, "degenerate bounds interval");
    if (!(blo <= tlo && thi <= bhi)) fail(CHEBFD_ERR_INVALID_ARGUMENT, "target outside bounds");
    if (degree < 1) fail(CHEBFD_ERR_INVALID_ARGUMENT, "window_coeffs: degree must be >= 1");
    const double alpha = 2.0 / (bhi - blo);
    const double beta = (blo + bhi) / (blo - bhi);
    auto clamp1 = [](double x) { return x < -1.0 ? -1.0 : (x > 1.0 ? 1.0 : x); };
    const double a_lo = std::acos(clamp1(alpha * tlo + beta));
    const double a_hi = std::acos(clamp1(alpha * thi + beta));
    std::vector<double> c(static_cast<size_t>(degree) + 1);
    c[0] = (a_lo - a_hi) / kPi;
    for (int n = 1; n <= degree; ++n)
        c[n] = 2.0 / (kPi * n) * (std::sin(n * a_lo) - std::sin(n * a_hi));
    return c;
}

// kernel_coeffs (filter.cpp:58-84)
std::vector<double> kernel_coeffs(int kind, int mu, int degree) {
    if (degree < 1) fail(CHEBFD_ERR_INVALID_ARGUMENT, "kernel_coeffs: degree must be >= 1");
    const int np = degree;
    std::vector<double> g(static_cast<size_t>(np) + 1, 1.0);
    switch (kind) {
        case CHEBFD_KERNEL_NONE: break;
        case CHEBFD_KERNEL_FEJER:
            for (int n = 0; n <= np; ++n) g[n] = static_cast<double>(np - n + 1) / (np + 1);
            break;
        case CHEBFD_KERNEL_JACKSON: {
            const double cot = std::cos(kPi / np) / std::sin(kPi / np);
            for (int n = 0; n <= np; ++n)
                g[n] = ((np - n) * std::cos(kPi * n / np) + std::sin(kPi * n / np) * cot) / np;
            break;
        }
        case CHEBFD_KERNEL_LANCZOS:
            if (mu < 1) fail(CHEBFD_ERR_INVALID_ARGUMENT, "lanczos kernel needs mu >= 1");
            for (int n = 1; n <= np; ++n) {
                const double x = kPi * n / (np + 1);
                g[n] = std::pow(std::sin(x) / x, mu);
            }
            break;
        default: fail(CHEBFD_ERR_INVALID_ARGUMENT, "unknown kernel");
    }
    return g;
}

// ChebSeriesDensity::count with Jackson damping (spectral.cpp:20-29,46-57)
double dos_count(const double* mu, int order, double blo, double bhi, double lo, double hi) {
    if (order < 0) fail(CHEBFD_ERR_INVALID_ARGUMENT, "ChebSeriesDensity: no moments");
    if (!(blo < bhi)) fail(CHEBFD_ERR_INVALID_ARGUMENT, "ChebSeriesDensity: bad bounds");
    if (hi < lo) return -dos_count(mu, order, blo, bhi, hi, lo);
    const double alpha = 2.0 / (bhi - blo);
    const double beta = (blo + bhi) / (blo - bhi);
    const auto g = kernel_coeffs(CHEBFD_KERNEL_JACKSON, 0, std::max(order, 1));
    std::vector<double> damped(static_cast<size_t>(order) + 1);
    for (int n = 0; n <= order; ++n) damped[n] = g[n] * mu[n];
    auto theta = [&](double l) { return std::acos(std::clamp(alpha * l + beta, -1.0, 1.0)); };
    const double th_lo = theta(lo), th_hi = theta(hi);
    double acc = damped[0] * (th_lo - th_hi);
    for (int n = 1; n <= order; ++n)
        acc += 2.0 * damped[n] * (std::sin(n * th_lo) - std::sin(n * th_hi)) / static_cast<double>(n);
    return acc / kPi;
}

// ChebSeriesDensity::density (spectral.cpp:31-44): Jackson-damped reconstruction at lambda
double dos_density(const double* mu, int order, double blo, double bhi, double lambda) {
    if (order < 0) fail(CHEBFD_ERR_INVALID_ARGUMENT, "ChebSeriesDensity: no moments");
    if (!(blo < bhi)) fail(CHEBFD_ERR_INVALID_ARGUMENT, "ChebSeriesDensity: bad bounds");
    const double alpha = 2.0 / (bhi - blo);
    const double beta = (blo + bhi) / (blo - bhi);
    const auto g = kernel_coeffs(CHEBFD_KERNEL_JACKSON, 0, std::max(order, 1));
    double x = alpha * lambda + beta;
    x = std::clamp(x, -1.0 + 1e-12, 1.0 - 1e-12);
    double acc = g[0] * mu[0];
    double tm2 = 1.0, tm1 = x;
    if (order >= 1) acc += 2.0 * (g[1] * mu[1]) * x;
    for (int n = 2; n <= order; ++n) {
        const double tn = 2.0 * x * tm1 - tm2;
        acc += 2.0 * (g[n] * mu[n]) * tn;
        tm2 = tm1;
        tm1 = tn;
    }
    return alpha * acc / (kPi * std::sqrt(1.0 - x * x));
}

void plane_partition(int64_t dim, int64_t plane, int rank, int nranks, int64_t* r0, int64_t* r1) {
    const int64_t planes = plane > 0 ? dim / plane : dim;
    const int64_t unit = plane > 0 ? plane : 1;
    if (planes < nranks)
        fail(CHEBFD_ERR_UNSUPPORTED, "fewer lattice planes than ranks: cannot partition");
    const int64_t p0 = planes * rank / nranks, p1 = planes * (rank + 1) / nranks;
    *r0 = p0 * unit;
    *r1 = (rank == nranks - 1) ? dim : p1 * unit;
}

}  // namespace cfd
