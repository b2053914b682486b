// Filter design on the host: damping factor sigma, quality eta, the degree
// rule and the DOS-driven search margin (/root/reference/proj/src/
// filter_design.cpp).  Pure scalar math; the evaluation points, comparison
// order and library calls follow the reference so that the chosen degree is
// the reference's integer (pinned in tests/test_design.py against the
// compiled reference).
#include <algorithm>
#include <cmath>
#include <limits>
#include <numbers>
#include <thread>
#include <vector>

#include "capi_common.hpp"

namespace cfd {

namespace {

constexpr double kPi = std::numbers::pi;
constexpr double kInf = std::numeric_limits<double>::infinity();

// One kernel-damped window polynomial on [blo, bhi] (filter.cpp:86-99)
struct Poly {
    int degree;
    std::vector<double> c;  // combined g_n c_n
    double alpha, beta, blo, bhi;

    // eval_scalar (filter.cpp:101-114); x is always inside [blo, bhi] here
    double at(double x) const {
        const double t = alpha * x + beta;
        double tm2 = 1.0, tm1 = t;
        double acc = c[0] + c[1] * t;
        for (int n = 2; n <= degree; ++n) {
            const double tn = 2.0 * t * tm1 - tm2;
            acc += c[n] * tn;
            tm2 = tm1;
            tm1 = tn;
        }
        return acc;
    }
    double theta(double x) const { return std::acos(std::clamp(alpha * x + beta, -1.0, 1.0)); }
    double x_at(double th) const { return std::clamp((std::cos(th) - beta) / alpha, blo, bhi); }
    double mag(double th) const { return std::abs(at(x_at(th))); }
};

Poly build(double tlo, double thi, double blo, double bhi, int degree, int kind, int mu) {
    Poly p;
    p.degree = degree;
    const auto c = window_coeffs(tlo, thi, blo, bhi, degree);
    const auto g = kernel_coeffs(kind, mu, degree);
    p.c.resize(c.size());
    for (size_t n = 0; n < c.size(); ++n) p.c[n] = g[n] * c[n];
    p.alpha = 2.0 / (bhi - blo);
    p.beta = (blo + bhi) / (blo - bhi);
    p.blo = blo;
    p.bhi = bhi;
    return p;
}

// First index of the extremum of f(j) over j = 0..n (skipping points where
// f returns a negative value), exactly the serial scan's answer: threads scan
// contiguous index ranges, and the merge keeps the smaller index on ties.
// Parallel once n x degree is large (paper-scale degrees).
template <class F>
std::pair<long, double> arg_extremum(long n, int degree, bool maximize, const F& f) {
    auto scan = [&](long j0, long j1) {
        long bj = -1;
        double bf = 0.0;
        for (long j = j0; j < j1; ++j) {
            const double v = f(j);
            if (v < 0.0) continue;
            if (bj < 0 || (maximize ? v > bf : v < bf)) {
                bf = v;
                bj = j;
            }
        }
        return std::make_pair(bj, bf);
    };
    const long total = n + 1;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    if (hw == 1 || static_cast<double>(total) * degree < 4e6) return scan(0, total);
    const long parts = std::min<long>(hw, total);
    std::vector<std::pair<long, double>> res(static_cast<size_t>(parts));
    std::vector<std::thread> th;
    for (long q = 0; q < parts; ++q)
        th.emplace_back([&, q] { res[q] = scan(total * q / parts, total * (q + 1) / parts); });
    for (auto& t : th) t.join();
    std::pair<long, double> best{-1, 0.0};
    for (const auto& r : res) {  // ranges in increasing index order: strict comparison keeps the first
        if (r.first < 0) continue;
        if (best.first < 0 || (maximize ? r.second > best.second : r.second < best.second)) best = r;
    }
    return best;
}

// golden-section search for an extremum of |p| over theta in [lo, hi]
double golden(const Poly& p, double lo, double hi, bool maximize) {
    const double r = (std::sqrt(5.0) - 1.0) / 2.0;
    double a = lo, b = hi;
    double c = b - r * (b - a), d = a + r * (b - a);
    double fc = p.mag(c), fd = p.mag(d);
    for (int it = 0; it < 60 && (b - a) > 1e-13 * kPi; ++it) {
        if (maximize ? (fc > fd) : (fc < fd)) {
            b = d;
            d = c;
            fd = fc;
            c = b - r * (b - a);
            fc = p.mag(c);
        } else {
            a = c;
            c = d;
            fc = fd;
            d = a + r * (b - a);
            fd = p.mag(d);
        }
    }
    const double f = p.mag(0.5 * (a + b));
    return maximize ? std::max({f, p.mag(lo), p.mag(hi)}) : std::min({f, p.mag(lo), p.mag(hi)});
}

// max |p| over [lo, hi]: grid scan then golden refinement around the best cell
double scan_max(const Poly& p, double lo, double hi, long n) {
    if (!(hi > lo)) return p.mag(lo);
    const double step = (hi - lo) / static_cast<double>(n);
    const long best =
        arg_extremum(n, p.degree, true, [&](long j) { return p.mag(lo + step * j); }).first;
    return golden(p, std::max(lo, lo + step * (best - 1)), std::min(hi, lo + step * (best + 1)), true);
}

struct Cfg {
    double tlo, thi, dprime, blo, bhi;
    double slo() const { return tlo - dprime; }
    double shi() const { return thi + dprime; }
    void validate() const {  // IntervalConfig::validate (filter_design.cpp:170-176)
        if (!(tlo < thi)) fail(CHEBFD_ERR_INVALID_ARGUMENT, "IntervalConfig: degenerate target");
        if (!(dprime > 0.0)) fail(CHEBFD_ERR_INVALID_ARGUMENT, "IntervalConfig: delta' must be > 0");
        if (!(blo < slo() && shi() < bhi))
            fail(CHEBFD_ERR_INVALID_ARGUMENT,
                 "IntervalConfig: search interval not strictly inside bounds");
    }
};

// sigma = max outside the search interval / min inside the target
// (filter_design.cpp:88-147,178-184)
double sigma_of(const Poly& p, const Cfg& cfg) {
    cfg.validate();
    const double th_s_hi = p.theta(cfg.shi()), th_s_lo = p.theta(cfg.slo());
    const double th_t_lo = p.theta(cfg.tlo), th_t_hi = p.theta(cfg.thi);
    // coarse grid in theta, points inside the search interval skipped
    const long m = std::max<long>(10L * p.degree, 2000);
    const double h = kPi / static_cast<double>(m);
    const long best_j = arg_extremum(m, p.degree, true, [&](long j) {
                            const double th = h * j;
                            if (th > th_s_hi && th < th_s_lo) return -1.0;  // inside I_S: skipped
                            return std::abs(p.at(p.x_at(th)));
                        }).first;
    const double best_th = best_j >= 0 ? h * best_j : 0.0;
    double lo = best_th - h, hi = best_th + h;
    if (best_th <= th_s_hi) {
        lo = std::max(lo, 0.0);
        hi = std::min(hi, th_s_hi);
    } else {
        lo = std::max(lo, th_s_lo);
        hi = std::min(hi, kPi);
    }
    double out = golden(p, lo, hi, true);
    // the lobes adjacent to the search-interval edges, densely
    const double lobe = kPi / static_cast<double>(std::max(p.degree, 1));
    out = std::max(out, scan_max(p, std::max(0.0, th_s_hi - 2.0 * lobe), th_s_hi, 256));
    out = std::max(out, scan_max(p, th_s_lo, std::min(kPi, th_s_lo + 2.0 * lobe), 256));
    // minimum over the target interval
    const double span = th_t_lo - th_t_hi;
    const long mt = std::max<long>(200, static_cast<long>(10.0 * p.degree * span / kPi) + 1);
    const long bmin = arg_extremum(mt, p.degree, false, [&](long j) {
                          return std::abs(p.at(p.x_at(th_t_hi + span * j / mt)));
                      }).first;
    const double ht = span / mt;
    const double a = std::max(th_t_hi, th_t_hi + ht * (static_cast<double>(bmin) - 1));
    const double b = std::min(th_t_lo, th_t_hi + ht * (static_cast<double>(bmin) + 1));
    const double in = golden(p, a, b, false);
    if (in < 1e-300) fail(CHEBFD_ERR_RUNTIME, "damping_factor: filter vanishes on the target interval");
    return out / in;
}

double eta_or_inf(const Cfg& cfg, int kind, int mu, int degree) {
    const Poly p = build(cfg.tlo, cfg.thi, cfg.blo, cfg.bhi, degree, kind, mu);
    const double s = sigma_of(p, cfg);
    return s >= 1.0 ? kInf : -static_cast<double>(degree) / std::log10(s);
}

double seed_constant(int kind) {  // filter_design.cpp:158-166
    switch (kind) {
        case CHEBFD_KERNEL_NONE: return 1.5;
        case CHEBFD_KERNEL_FEJER: return 4.0;
        case CHEBFD_KERNEL_JACKSON: return 7.0;
        case CHEBFD_KERNEL_LANCZOS: return 6.2;
    }
    return 6.0;
}

}  // namespace

double quality_of(int degree, double sigma) {  // filter_design.cpp:186-190
    if (!(sigma > 0.0)) fail(CHEBFD_ERR_DOMAIN, "quality: sigma must be positive");
    if (sigma >= 1.0) fail(CHEBFD_ERR_DOMAIN, "quality: sigma >= 1, filter does not damp");
    return -static_cast<double>(degree) / std::log10(sigma);
}

double damping_factor(double tlo, double thi, double dprime, double blo, double bhi, int degree,
                      int kind, int mu) {
    const Cfg cfg{tlo, thi, dprime, blo, bhi};
    cfg.validate();
    return sigma_of(build(tlo, thi, blo, bhi, degree, kind, mu), cfg);
}

// optimize_degree (filter_design.cpp:204-277)
DesignOut optimize_degree(double tlo, double thi, double dprime, double blo, double bhi, int kind,
                          int mu, double epsilon) {
    const Cfg cfg{tlo, thi, dprime, blo, bhi};
    cfg.validate();
    if (!(epsilon > 0.0 && epsilon < 1.0))
        fail(CHEBFD_ERR_INVALID_ARGUMENT, "optimize_degree: epsilon must be in (0,1)");
    const double seed = seed_constant(kind) * (0.5 * (bhi - blo)) / dprime;
    int best = 0, rising = 0, prev = 0;
    double best_eta = kInf;
    // geometric walk (ratio 1.1) from below the seed until clearly past the minimum
    for (double g = std::max(4.0, seed / 8.0); g <= seed * 16.0; g *= 1.1) {
        const int np = std::max(prev + 1, static_cast<int>(std::lround(g)));
        prev = np;
        const double eta = eta_or_inf(cfg, kind, mu, np);
        if (eta < best_eta) {
            best_eta = eta;
            best = np;
            rising = 0;
        } else if (std::isfinite(best_eta)) {
            ++rising;
            if (rising >= 4 && np > seed && eta > 1.2 * best_eta) break;
        }
    }
    if (!std::isfinite(best_eta))
        fail(CHEBFD_ERR_RUNTIME, "optimize_degree: no degree with sigma < 1 in search range");
    // integer refinement of the bracketing cells (9 samples per pass)
    int lo = std::max(2, static_cast<int>(std::lround(best / 1.1)));
    int hi = static_cast<int>(std::lround(best * 1.1));
    while (hi - lo > 2) {
        std::vector<int> pts;
        int arg = lo, last = -1;
        double arg_eta = kInf;
        for (int j = 0; j <= 9; ++j) {
            const int np = lo + static_cast<int>(std::lround(static_cast<double>(hi - lo) * j / 9));
            if (np == last) continue;
            last = np;
            pts.push_back(np);
            const double eta = eta_or_inf(cfg, kind, mu, np);
            if (eta < arg_eta) {
                arg_eta = eta;
                arg = np;
            }
        }
        best = arg;
        best_eta = arg_eta;
        const auto it = std::find(pts.begin(), pts.end(), arg);
        const int nlo = it == pts.begin() ? *it : *(it - 1);
        const int nhi = it + 1 == pts.end() ? *it : *(it + 1);
        if (nhi - nlo >= hi - lo) break;
        lo = nlo;
        hi = nhi;
    }
    for (int np = lo; np <= hi; ++np) {
        const double eta = eta_or_inf(cfg, kind, mu, np);
        if (eta < best_eta) {
            best_eta = eta;
            best = np;
        }
    }
    DesignOut r;
    r.np_opt = best;
    r.sigma = sigma_of(build(tlo, thi, blo, bhi, best, kind, mu), cfg);
    r.eta_opt = quality_of(best, r.sigma);
    r.predicted_mvms = r.eta_opt * (-std::log10(epsilon));
    r.predicted_iters = static_cast<int>(std::ceil(std::log10(epsilon) / std::log10(r.sigma)));
    r.delta_prime = dprime;
    return r;
}

// invert_search_margin (filter_design.cpp:330-354): bisection on the DOS count
double invert_search_margin(const double* mu, int order, double blo, double bhi, double tlo,
                            double thi, double n_search) {
    if (!(blo <= tlo && thi <= bhi))
        fail(CHEBFD_ERR_INVALID_ARGUMENT, "invert_search_margin: target outside DOS bounds");
    const double n_target = dos_count(mu, order, blo, bhi, tlo, thi);
    if (n_search <= n_target) fail(CHEBFD_ERR_RUNTIME, "invert_search_margin: N_S <= estimated N_T (pole)");
    const double dmax = 0.999 * std::min(tlo - blo, bhi - thi);
    auto count_at = [&](double d) { return dos_count(mu, order, blo, bhi, tlo - d, thi + d); };
    double lo = 0.0, hi = dmax;
    if (count_at(dmax) < n_search)
        fail(CHEBFD_ERR_RUNTIME, "invert_search_margin: search space exceeds available spectrum");
    for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        const double f = count_at(mid) - n_search;
        if (std::abs(f) <= 1e-6 * n_search || (hi - lo) < 1e-15 * dmax) {
            lo = hi = mid;
            break;
        }
        (f < 0.0 ? lo : hi) = mid;
    }
    return 0.5 * (lo + hi);
}

// choose_parameters (filter_design.cpp:356-369)
DesignOut choose_parameters(const double* mu, int order, double blo, double bhi, double tlo,
                            double thi, double n_search, int kind, int kmu, double epsilon) {
    const double n_target = dos_count(mu, order, blo, bhi, tlo, thi);
    if (n_target < 0.5) fail(CHEBFD_ERR_RUNTIME, "choose_parameters: empty target interval");
    const double dp = invert_search_margin(mu, order, blo, bhi, tlo, thi, n_search);
    DesignOut out = optimize_degree(tlo, thi, dp, blo, bhi, kind, kmu, epsilon);
    out.n_target_estimate = n_target;
    out.below_recommended = n_search < std::ceil(1.25 * n_target);
    return out;
}

}  // namespace cfd

using namespace cfd;

extern "C" {

int chebfd_damping_factor(double tlo, double thi, double delta_prime, double blo, double bhi,
                          int degree, int kernel, int mu, double* sigma) {
    return guard([&] { *sigma = damping_factor(tlo, thi, delta_prime, blo, bhi, degree, kernel, mu); });
}

int chebfd_optimize_degree(double tlo, double thi, double delta_prime, double blo, double bhi,
                           int kernel, int mu, double epsilon, chebfd_design* out) {
    return guard([&] {
        const DesignOut d = optimize_degree(tlo, thi, delta_prime, blo, bhi, kernel, mu, epsilon);
        out->np_opt = d.np_opt;
        out->eta_opt = d.eta_opt;
        out->sigma = d.sigma;
        out->predicted_mvms = d.predicted_mvms;
        out->predicted_iters = d.predicted_iters;
        out->delta_prime = d.delta_prime;
        out->n_target_estimate = 0.0;
        out->below_recommended_search_space = 0;
    });
}

int chebfd_choose_parameters(const double* mu, int order, double blo, double bhi, double tlo,
                             double thi, double n_search, int kernel, int kmu, double epsilon,
                             chebfd_design* out) {
    return guard([&] {
        const DesignOut d =
            choose_parameters(mu, order, blo, bhi, tlo, thi, n_search, kernel, kmu, epsilon);
        out->np_opt = d.np_opt;
        out->eta_opt = d.eta_opt;
        out->sigma = d.sigma;
        out->predicted_mvms = d.predicted_mvms;
        out->predicted_iters = d.predicted_iters;
        out->delta_prime = d.delta_prime;
        out->n_target_estimate = d.n_target_estimate;
        out->below_recommended_search_space = d.below_recommended ? 1 : 0;
    });
}

int chebfd_invert_search_margin(const double* mu, int order, double blo, double bhi, double tlo,
                                double thi, double n_search, double* delta_prime) {
    return guard([&] { *delta_prime = invert_search_margin(mu, order, blo, bhi, tlo, thi, n_search); });
}

}  // extern "C"
