// ChebFD driver on the device: SVQB (solver.cpp:32-61), Rayleigh-Ritz
// (:63-91), Lanczos bounds (spectral.cpp:96-154), stochastic KPM DOS
// (spectral.cpp:156-205) and the outer loop solve() (solver.cpp:93-214).
// The host runs the reference's control flow; every O(D) operation is a
// device kernel on the context stream; only n_b x n_b matrices and n_b-length
// vectors cross PCIe.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

#include "capi_common.hpp"

namespace cfd {

namespace {

using Cx = std::complex<double>;

// host copy of a small S-valued matrix
struct Small {
    int kind;
    int64_t rows, cols;
    std::vector<double> a;  // interleaved if complex
    Small(int k, int64_t r, int64_t c) : kind(k), rows(r), cols(c), a(static_cast<size_t>(r * c) * (k ? 2 : 1), 0.0) {}
    double& re(int64_t i, int64_t j) { return a[(kind ? 2 : 1) * static_cast<size_t>(i * cols + j)]; }
    double& im(int64_t i, int64_t j) { return a[2 * static_cast<size_t>(i * cols + j) + 1]; }
};

// ge = 0.5 (G + G^H) as Eigen evaluates S(0.5) * (ge + ge.adjoint()) (solver.cpp:37,69)
void symmetrize(Small& g) {
    const int64_t n = g.rows;
    Small out = g;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) {
            if (g.kind) {
                const Cx s = Cx(g.re(i, j), g.im(i, j)) + std::conj(Cx(g.re(j, i), g.im(j, i)));
                const Cx r = Cx(0.5) * s;
                out.re(i, j) = r.real();
                out.im(i, j) = r.imag();
            } else {
                out.re(i, j) = 0.5 * (g.re(i, j) + g.re(j, i));
            }
        }
    g = out;
}

struct SvqbOut {
    std::unique_ptr<Block> q;
    int64_t rank = 0;
};

// svqb_orthonormalize (solver.cpp:32-61); q has `rank` columns
SvqbOut svqb(Context& c, const Matrix* shape, Block& y, double drop_tol) {
    const int64_t nb = y.width;
    if (nb < 1) fail(CHEBFD_ERR_INVALID_ARGUMENT, "svqb: empty block");
    Small g(y.kind, nb, nb);
    gram_host(c, y, y, g.a.data());
    symmetrize(g);
    std::vector<double> lam(nb);
    Small v(y.kind, nb, nb);
    if (!heev_host(c, y.kind, nb, g.a.data(), lam.data(), v.a.data(), true))
        fail(CHEBFD_ERR_RUNTIME, "svqb: Gram eigensolve failed");
    const double lmax = lam[nb - 1];
    double trace = 0.0;
    for (double l : lam) trace += l;
    if (lam[0] < -1e-12 * std::max(trace, 0.0))
        fail(CHEBFD_ERR_RUNTIME, "svqb: Gram matrix indefinite, corrupted input");
    std::vector<int64_t> keep;
    for (int64_t i = 0; i < nb; ++i)
        if (lam[i] > drop_tol * lmax && lam[i] > 0.0) keep.push_back(i);
    if (keep.empty()) fail(CHEBFD_ERR_RUNTIME, "svqb: block numerically zero");
    const int64_t r = static_cast<int64_t>(keep.size());
    Small cm(y.kind, nb, r);
    for (int64_t j = 0; j < r; ++j) {
        const double s = std::sqrt(lam[keep[j]]);
        for (int64_t i = 0; i < nb; ++i) {
            cm.re(i, j) = v.re(i, keep[j]) / s;
            if (y.kind) cm.im(i, j) = v.im(i, keep[j]) / s;
        }
    }
    SvqbOut out;
    out.q = make_block(c, shape, y.kind, y.rows, r, false);
    mult_small_host_b(c, y, cm.a.data(), r, *out.q);
    out.rank = r;
    return out;
}

struct Ritz {
    std::vector<double> values, res;
    std::unique_ptr<Block> vectors;
};

// rayleigh_ritz (solver.cpp:63-91)
Ritz rayleigh_ritz(Context& c, const Matrix& a, Block& q) {
    const int64_t nb = q.width;
    auto aq = make_block(c, &a, q.kind, q.rows, nb, false);
    StepArgs s{};
    s.kind_step = kStepSpmmvm;
    s.w = aq->owned();
    s.alpha = 1.0;
    s.beta = 0.0;
    run_step_all(c, a, s, q);
    Small p(q.kind, nb, nb);
    // P = Q^H (A Q) is Hermitian (A Hermitian): its upper half suffices; symmetrize keeps
    // the reference's P = (G + G^H) / 2 (solver.cpp:68-70) for non-Hermitian input
    gram_host(c, q, *aq, p.a.data(), a.hermitian);
    symmetrize(p);
    Ritz out;
    out.values.resize(nb);
    Small rot(q.kind, nb, nb);
    if (!heev_host(c, q.kind, nb, p.a.data(), out.values.data(), rot.a.data(), true))
        fail(CHEBFD_ERR_RUNTIME, "rayleigh_ritz: projected eigensolve failed");
    out.vectors = make_block(c, &a, q.kind, q.rows, nb, false);
    auto av = make_block(c, &a, q.kind, q.rows, nb, false);
    DeviceBuffer& drot = c.small[0];
    drot.ensure(std::max<size_t>(rot.a.size() * sizeof(double), 16));
    CFD_CUDA(cudaMemcpyAsync(drot.p, rot.a.data(), rot.a.size() * sizeof(double),
                             cudaMemcpyHostToDevice, c.stream));
    mult_small_dev_b(c, q, drot.p, nb, *out.vectors);
    mult_small_dev_b(c, *aq, drot.p, nb, *av);
    // residual norms ||A v_k - lambda_k v_k|| fused into one reduction pass
    DeviceBuffer& dlam = c.small[1];
    dlam.ensure(sizeof(double) * std::max<int64_t>(nb, 1));
    CFD_CUDA(cudaMemcpyAsync(dlam.p, out.values.data(), sizeof(double) * nb, cudaMemcpyHostToDevice,
                             c.stream));
    c.dscratch.ensure(sizeof(double) * nb);
    launch_residual_sq(c, *av, *out.vectors, dlam.as<double>(), c.dscratch.p, c.stream);
    allreduce_sum(c, c.dscratch.as<double>(), nb, c.stream);
    out.res.resize(nb);
    CFD_CUDA(cudaMemcpyAsync(out.res.data(), c.dscratch.p, sizeof(double) * nb,
                             cudaMemcpyDeviceToHost, c.stream));
    ctx_sync(c);
    for (auto& r : out.res) r = std::sqrt(r);
    return out;
}

void divide_columns(Context& c, Block& b, const std::vector<double>& d) {
    DeviceBuffer& dd = c.small[1];
    dd.ensure(sizeof(double) * std::max<size_t>(d.size(), 1));
    CFD_CUDA(cudaMemcpyAsync(dd.p, d.data(), sizeof(double) * d.size(), cudaMemcpyHostToDevice,
                             c.stream));
    launch_scale_columns(c, b, dd.as<double>(), c.stream);
    ctx_sync(c);
}

std::vector<double> norms(Context& c, const Block& x) {
    std::vector<double> d(static_cast<size_t>(x.width) * (x.kind ? 2 : 1));
    column_dots_host(c, x, x, d.data());
    std::vector<double> n(x.width);
    for (int64_t k = 0; k < x.width; ++k) n[k] = std::sqrt(x.kind ? d[2 * k] : d[k]);
    return n;
}

void randomize(Context& c, Block& b, uint64_t seed) { randomize_upload(c, b, seed); }

// symmetric tridiagonal eigenvalues (Lanczos T) via cuSOLVER
std::vector<double> tridiag_eigs(Context& c, const std::vector<double>& al,
                                 const std::vector<double>& be) {
    const int64_t k = static_cast<int64_t>(al.size());
    std::vector<double> t(static_cast<size_t>(k * k), 0.0), w(k);
    for (int64_t j = 0; j < k; ++j) {
        t[j * k + j] = al[j];
        if (j + 1 < k) t[j * k + j + 1] = t[(j + 1) * k + j] = be[j];
    }
    if (!heev_host(c, CHEBFD_REAL64, k, t.data(), w.data(), nullptr, false))
        fail(CHEBFD_ERR_RUNTIME, "lanczos_bounds: tridiagonal eigensolve failed");
    return w;
}

}  // namespace

// lanczos_bounds (spectral.cpp:96-154)
void lanczos_bounds(Context& c, const Matrix& a, int iters, uint64_t seed, double* lo, double* hi) {
    if (iters < 2) fail(CHEBFD_ERR_INVALID_ARGUMENT, "lanczos_bounds: iters must be >= 2");
    const int64_t d = a.part.dim;
    const int m = static_cast<int>(std::min<int64_t>(iters, d));
    for (int restart = 0; restart < 4; ++restart) {
        auto v = make_block(c, &a, a.kind, a.part.local, 1, false);
        randomize(c, *v, seed + 977 * restart);
        divide_columns(c, *v, norms(c, *v));
        std::vector<std::unique_ptr<Block>> basis;
        std::vector<double> al, be;
        bool breakdown = false;
        for (int j = 0; j < m; ++j) {
            basis.push_back(std::move(v));
            Block& last = *basis.back();
            auto w = make_block(c, &a, a.kind, a.part.local, 1, false);
            StepArgs s{};
            s.kind_step = kStepSpmmvm;
            s.w = w->owned();
            s.alpha = 1.0;
            s.beta = 0.0;
            run_step_all(c, a, s, last);
            // full reorthogonalisation against all previous basis vectors
            for (int pass = 0; pass < 2; ++pass)
                for (auto& q : basis) {
                    double h[2] = {0.0, 0.0};
                    column_dots_host(c, *q, *w, h);
                    launch_axpy_scalar(c, *w, *q, h[0], a.kind ? h[1] : 0.0, c.stream);
                    if (pass == 0 && q.get() == &last) al.push_back(h[0]);
                }
            const double b_j = norms(c, *w)[0];
            if (j + 1 == m || static_cast<int64_t>(basis.size()) == d) break;
            if (b_j < 1e-14) {
                breakdown = true;
                break;
            }
            be.push_back(b_j);
            divide_columns(c, *w, {b_j});
            v = std::move(w);
        }
        if (breakdown && al.size() < 2 && restart < 3) continue;
        if (al.empty()) continue;
        const auto ev = tridiag_eigs(c, al, be);
        const double rmin = *std::min_element(ev.begin(), ev.end());
        const double rmax = *std::max_element(ev.begin(), ev.end());
        const double pad = 0.01 * (rmax - rmin) + 1e-12 * (1.0 + std::abs(rmin) + std::abs(rmax));
        *lo = rmin - pad;
        *hi = rmax + pad;
        return;
    }
    fail(CHEBFD_ERR_RUNTIME, "lanczos_bounds: repeated breakdown");
}

// kpm_dos (spectral.cpp:156-205): raw moments mu[0..order]
std::vector<double> kpm_dos(Context& c, const Matrix& a, double blo, double bhi, int order,
                            int samples, uint64_t seed) {
    if (order < 2) fail(CHEBFD_ERR_INVALID_ARGUMENT, "kpm_dos: order must be >= 2");
    if (samples < 1) fail(CHEBFD_ERR_INVALID_ARGUMENT, "kpm_dos: need at least one sample");
    const int64_t d = a.part.dim;
    const double alpha = 2.0 / (bhi - blo);
    const double beta = (blo + bhi) / (blo - bhi);
    auto z = make_block(c, &a, a.kind, a.part.local, samples, false);
    randomize(c, *z, seed);
    divide_columns(c, *z, norms(c, *z));
    auto u = make_block(c, &a, a.kind, a.part.local, samples, false);
    auto w = make_block(c, &a, a.kind, a.part.local, samples, false);
    const int nchecks = order / 128;
    // doubling: recurrence step n (V_n from V_n-1) yields the raw sums of moments 2n-2 and
    // 2n-1 (<V_n-1, V_n-1>, <V_n-1, V_n>), so order/2 + 1 steps give all order + 1 moments
    const bool dbl = moment_doubling(c, a);
    const int last_step = dbl ? order / 2 + 1 : order;
    DeviceBuffer mom(sizeof(double) * (order + 3) * samples);
    const size_t nrm_row = static_cast<size_t>(samples) * (a.kind ? 2 : 1);
    DeviceBuffer nrm(sizeof(double) * std::max<size_t>(nrm_row * nchecks, 1));
    // u = h z; w = z (x0 copy); dots rows 0 (<z,z>), 1 (<z,u>)
    StepArgs s{};
    s.kind_step = kStepSpmmvm;
    s.w = u->owned();
    s.x0 = w->owned();
    s.alpha = alpha;
    s.beta = beta;
    s.dots_mode = 3;
    s.dots_out = mom.p;
    run_step_all(c, a, s, *z);
    Block* pu = u.get();
    Block* pw = w.get();
    for (int n = 2; n <= last_step; ++n) {
        if (n > 2) std::swap(pu, pw);
        StepArgs r{};
        r.kind_step = kStepRecur;
        r.w = pw->owned();
        r.x0 = dbl ? nullptr : z->owned();
        r.alpha = 2.0 * alpha;
        r.beta = 2.0 * beta;
        r.dots_mode = dbl ? 4 : 2;
        r.dots_out = mom.as<double>() + static_cast<int64_t>(dbl ? 2 * n - 2 : n) * samples;
        run_step_all(c, a, r, *pu);
        if (n % 128 == 0)
            launch_column_reduce(c, *pw, *pw, 0, nrm.as<double>() + (n / 128 - 1) * nrm_row, c.stream);
    }
    allreduce_sum(c, mom.as<double>(), static_cast<size_t>(order + 1) * samples, c.stream);
    if (nchecks) allreduce_sum(c, nrm.as<double>(), nrm_row * nchecks, c.stream);
    std::vector<double> hm(static_cast<size_t>(order + 1) * samples), hn(nrm_row * nchecks);
    CFD_CUDA(cudaMemcpyAsync(hm.data(), mom.p, hm.size() * sizeof(double), cudaMemcpyDeviceToHost,
                             c.stream));
    if (nchecks)
        CFD_CUDA(cudaMemcpyAsync(hn.data(), nrm.p, hn.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                 c.stream));
    ctx_sync(c);
    if (dbl) moments_from_doubling(hm.data(), order + 1, samples);
    const double scale = static_cast<double>(d) / samples;
    std::vector<double> mu(static_cast<size_t>(order) + 1, 0.0);
    mu[0] = static_cast<double>(d);
    for (int n = 1; n <= order; ++n) {
        double sum = 0.0;
        for (int k = 0; k < samples; ++k) sum += hm[static_cast<size_t>(n) * samples + k];
        mu[n] = scale * sum;
        if (!std::isfinite(mu[n]) || std::abs(mu[n]) > 4.0 * d)
            fail(CHEBFD_ERR_RUNTIME, "kpm_dos: moment growth indicates spectrum outside bounds");
        if (n % 128 == 0 && n <= last_step) {
            for (int k = 0; k < samples; ++k) {
                const double v = std::sqrt(hn[(n / 128 - 1) * nrm_row + (a.kind ? 2 * k : k)]);
                if (!std::isfinite(v) || v > 4.0)
                    fail(CHEBFD_ERR_RUNTIME, "kpm_dos: recurrence growth, bounds violated");
            }
        }
    }
    return mu;
}

}  // namespace cfd

using namespace cfd;

extern "C" {

int chebfd_svqb(chebfd_block* y, double drop_tol, chebfd_block* q, int64_t* rank) {
    return guard([&] {
        Block& Y = *reinterpret_cast<Block*>(y);
        Block& Q = *reinterpret_cast<Block*>(q);
        check_same_shape(Y, Q);
        auto r = svqb(*Y.ctx, Y.shape_of, Y, drop_tol);
        CFD_CUDA(cudaMemsetAsync(Q.buf.p, 0, Q.buf.bytes, Y.ctx->stream));
        launch_copy_columns(*Y.ctx, Q, 0, *r.q, 0, r.rank, Y.ctx->stream);
        ctx_sync(*Y.ctx);
        *rank = r.rank;
    });
}

int chebfd_rayleigh_ritz(chebfd_matrix* a, chebfd_block* q, chebfd_block* v, double* values,
                         double* residual_norms) {
    return guard([&] {
        Matrix& m = *reinterpret_cast<Matrix*>(a);
        Block& Q = *reinterpret_cast<Block*>(q);
        Block& V = *reinterpret_cast<Block*>(v);
        check_conforms(m, Q, "rayleigh_ritz");
        check_same_shape(Q, V);
        Ritz r = rayleigh_ritz(*m.ctx, m, Q);
        CFD_CUDA(cudaMemcpyAsync(V.owned(), r.vectors->owned(), V.owned_bytes(),
                                 cudaMemcpyDeviceToDevice, m.ctx->stream));
        ctx_sync(*m.ctx);
        std::memcpy(values, r.values.data(), sizeof(double) * r.values.size());
        std::memcpy(residual_norms, r.res.data(), sizeof(double) * r.res.size());
    });
}

int chebfd_lanczos_bounds(chebfd_matrix* a, int iters, uint64_t seed, double* lo, double* hi) {
    return guard([&] {
        Matrix& m = *reinterpret_cast<Matrix*>(a);
        lanczos_bounds(*m.ctx, m, iters, seed, lo, hi);
    });
}

int chebfd_kpm_dos(chebfd_matrix* a, double blo, double bhi, int order, int samples, uint64_t seed,
                   double* mu) {
    return guard([&] {
        Matrix& m = *reinterpret_cast<Matrix*>(a);
        auto v = kpm_dos(*m.ctx, m, blo, bhi, order, samples, seed);
        std::memcpy(mu, v.data(), sizeof(double) * v.size());
    });
}

int chebfd_dos_count(const double* mu, int order, double blo, double bhi, double lo, double hi,
                     double* out) {
    return guard([&] { *out = dos_count(mu, order, blo, bhi, lo, hi); });
}

void chebfd_solver_options_default(chebfd_solver_options* o) {
    // SolverOptions defaults (solver.hpp:12-25)
    o->target_lo = o->target_hi = 0.0;
    o->epsilon = 1e-10;
    o->n_search = 0;
    o->degree = 0;
    o->kernel = CHEBFD_KERNEL_LANCZOS;
    o->kernel_mu = 2;
    o->max_iters = 40;
    o->seed = 1;
    o->dos_moments = 2000;
    o->dos_samples = 32;
    o->bounds_lo = o->bounds_hi = 0.0;
    o->collect_weight_density = 1;
}

int chebfd_dos_density(const double* mu, int order, double blo, double bhi, double lambda,
                       double* out) {
    return guard([&] { *out = dos_density(mu, order, blo, bhi, lambda); });
}

int chebfd_weight_density(const double* moments, int degree, int64_t width, double* mu) {
    return guard([&] {
        // weight_density (spectral.cpp:81-88): mu[n] = sum_k m(n, k), k in column order
        if (width <= 0 || degree < 0 || moments == nullptr)
            fail(CHEBFD_ERR_INVALID_ARGUMENT, "weight_density: empty moment table");
        for (int n = 0; n <= degree; ++n) {
            double acc = 0.0;
            for (int64_t k = 0; k < width; ++k) acc += moments[static_cast<int64_t>(n) * width + k];
            mu[n] = acc;
        }
    });
}

int chebfd_solve(chebfd_matrix* a, const chebfd_solver_options* o, chebfd_solve_report* rep,
                 int cap, double* values, double* residual_norms, int* accepted, double* history,
                 chebfd_block** vectors) {
    return chebfd_solve_ex(a, o, rep, cap, values, residual_norms, accepted, history, vectors, 0,
                           nullptr, nullptr);
}

int chebfd_solve_ex(chebfd_matrix* a, const chebfd_solver_options* o, chebfd_solve_report* rep,
                    int cap, double* values, double* residual_norms, int* accepted,
                    double* history, chebfd_block** vectors, int weight_cap,
                    double* weight_moments, int* weight_len) {
    return guard([&] {
        if (weight_len) *weight_len = 0;
        Matrix& A = *reinterpret_cast<Matrix*>(a);
        Context& c = *A.ctx;
        const auto t0 = std::chrono::steady_clock::now();
        if (o->epsilon <= 0.0) fail(CHEBFD_ERR_INVALID_ARGUMENT, "solve: epsilon must be positive");
        if (o->max_iters < 1) fail(CHEBFD_ERR_INVALID_ARGUMENT, "solve: max_iters must be >= 1");
        if (!(o->target_lo < o->target_hi))
            fail(CHEBFD_ERR_INVALID_ARGUMENT, "solve: degenerate target");
        std::memset(rep, 0, sizeof(*rep));
        using clk = std::chrono::steady_clock;
        auto secs = [](clk::time_point a) {
            return std::chrono::duration<double>(clk::now() - a).count();
        };
        auto tp = clk::now();
        // with N_S given, the start block (solver.cpp:147-154) does not depend on the DOS:
        // generate it on a helper thread while the device runs the bounds and the KPM DOS
        std::unique_ptr<Block> x_early;
        std::unique_ptr<AsyncRandomize> x_job;
        // (only for blocks whose generation takes longer than the helper's set-up: pinned
        // buffers and a stream cost ~50 ms, a C1 block takes 6 ms synchronously)
        if (o->n_search > 0 && c.async_start_entries > 0 &&
            A.part.local * o->n_search >= c.async_start_entries) {
            x_early = make_block(c, &A, A.kind, A.part.local, o->n_search, false);
            ctx_sync(c);  // the (cached) storage and its halo clear are settled on c.stream
            x_job = std::make_unique<AsyncRandomize>(c, *x_early, o->seed + 2);
        }
        double blo = o->bounds_lo, bhi = o->bounds_hi;
        if (!(blo < bhi)) lanczos_bounds(c, A, 30, o->seed, &blo, &bhi);
        rep->t_bounds = secs(tp);
        tp = clk::now();
        rep->bounds_lo = blo;
        rep->bounds_hi = bhi;
        rep->matrix_norm_est = std::max(std::abs(blo), std::abs(bhi));
        const auto mu = kpm_dos(c, A, blo, bhi, o->dos_moments, o->dos_samples, o->seed + 1);
        rep->t_dos = secs(tp);
        tp = clk::now();
        // estimate_count (spectral.cpp:90-94)
        if (!(blo <= o->target_lo && o->target_hi <= bhi))
            fail(CHEBFD_ERR_INVALID_ARGUMENT, "estimate_count: interval outside DOS bounds");
        rep->n_target_estimate =
            dos_count(mu.data(), o->dos_moments, blo, bhi, o->target_lo, o->target_hi);
        if (rep->n_target_estimate < 0.5) {  // empty target: immediate success
            rep->converged = 1;
            rep->seconds =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            return;
        }
        rep->n_search = o->n_search > 0 ? o->n_search
                                        : 2 * static_cast<int>(std::ceil(rep->n_target_estimate));
        if (o->degree > 0) {
            rep->degree = o->degree;
            // sigma / eta of the imposed degree, for reporting only (solver.cpp:114-129)
            try {
                const double dp = invert_search_margin(mu.data(), o->dos_moments, blo, bhi,
                                                       o->target_lo, o->target_hi, rep->n_search);
                rep->sigma = damping_factor(o->target_lo, o->target_hi, dp, blo, bhi, rep->degree,
                                            o->kernel, o->kernel_mu);
                rep->eta = rep->sigma < 1.0 ? quality_of(rep->degree, rep->sigma) : 0.0;
            } catch (const std::exception&) {
                rep->sigma = 0.0;
                rep->eta = 0.0;
            }
        } else {  // choose_parameters (solver.cpp:130-136)
            const DesignOut d = choose_parameters(mu.data(), o->dos_moments, blo, bhi, o->target_lo,
                                                  o->target_hi, rep->n_search, o->kernel,
                                                  o->kernel_mu, o->epsilon);
            rep->degree = d.np_opt;
            rep->sigma = d.sigma;
            rep->eta = d.eta_opt;
        }
        rep->t_design = secs(tp);
        if (rep->degree < 2) fail(CHEBFD_ERR_RUNTIME, "solve: filter degree must be >= 2");
        const int np = rep->degree;
        std::vector<double> combined(np + 1);
        double alpha = 0, beta = 0;
        {
            auto cc = window_coeffs(o->target_lo, o->target_hi, blo, bhi, np);
            auto gg = kernel_coeffs(o->kernel, o->kernel_mu, np);
            for (int n = 0; n <= np; ++n) combined[n] = gg[n] * cc[n];
            alpha = 2.0 / (bhi - blo);
            beta = (blo + bhi) / (blo - bhi);
        }
        const double sqrt_eps = std::sqrt(o->epsilon);
        const double required =
            std::max(1.0, std::ceil(rep->n_target_estimate - 3.0 * std::sqrt(rep->n_target_estimate)));
        const int64_t ns = rep->n_search;
        tp = clk::now();
        std::unique_ptr<Block> x;
        if (x_job && ns == x_early->width) {
            x_job->join();
            x = std::move(x_early);
        } else {
            if (x_job) x_job->join();
            x = make_block(c, &A, A.kind, A.part.local, ns, false);
            randomize(c, *x, o->seed + 2);
        }
        divide_columns(c, *x, norms(c, *x));  // unit columns (solver.cpp:149-154)
        rep->t_start = secs(tp);
        Ritz ritz;
        std::vector<double> mom;
        for (int iter = 1; iter <= o->max_iters; ++iter) {
            if (o->collect_weight_density) mom.assign(static_cast<size_t>(np + 1) * x->width, 0.0);
            tp = clk::now();
            apply_filter_device(c, A, *x, combined.data(), np, alpha, beta,
                                o->collect_weight_density ? mom.data() : nullptr);
            ctx_sync(c);
            rep->t_filter += secs(tp);
            tp = clk::now();
            if (o->collect_weight_density) {
                // rep.weight = weight_density(moments, bounds) of this iteration's filter
                // (solver.cpp:158-162, spectral.cpp:81-88): mu[n] = sum_k m(n, k)
                double w0 = 0.0;
                for (int64_t k = 0; k < x->width; ++k) w0 += mom[k];
                rep->weight_integral = w0;
                if (weight_moments) {
                    if (weight_cap < np + 1)
                        fail(CHEBFD_ERR_INVALID_ARGUMENT, "solve: weight capacity too small");
                    for (int n = 0; n <= np; ++n) {
                        double acc = 0.0;
                        for (int64_t k = 0; k < x->width; ++k) acc += mom[static_cast<size_t>(n) * x->width + k];
                        weight_moments[n] = acc;
                    }
                    if (weight_len) *weight_len = np + 1;
                }
            }
            SvqbOut ortho = svqb(c, &A, *x, 1e-14);
            for (int repair = 0; ortho.rank < ns && repair < 5; ++repair) {
                auto padded = make_block(c, &A, A.kind, A.part.local, ns, false);
                auto fresh = make_block(c, &A, A.kind, A.part.local, ns - ortho.rank, false);
                randomize(c, *fresh, o->seed + 1000 + iter * 13 + repair);
                launch_copy_columns(c, *padded, 0, *ortho.q, 0, ortho.rank, c.stream);
                launch_copy_columns(c, *padded, ortho.rank, *fresh, 0, ns - ortho.rank, c.stream);
                ortho = svqb(c, &A, *padded, 1e-14);
            }
            rep->t_ortho += secs(tp);
            tp = clk::now();
            ritz = rayleigh_ritz(c, A, *ortho.q);
            rep->t_rr += secs(tp);
            const int64_t nb = ritz.vectors->width;
            int acc = 0, pending = 0;
            double rmin = 0.0, rmax = 0.0;
            bool any = false;
            std::vector<int> acc_flags(nb, 0);
            for (int64_t k = 0; k < nb; ++k) {
                const double v = ritz.values[k];
                if (!(v >= o->target_lo && v <= o->target_hi)) continue;
                const double r = ritz.res[k];
                if (r > sqrt_eps) continue;  // ghost for this iteration
                if (r <= o->epsilon) {
                    acc_flags[k] = 1;
                    ++acc;
                } else {
                    ++pending;
                }
                if (!any || r < rmin) rmin = r;
                if (!any || r > rmax) rmax = r;
                any = true;
            }
            rep->iterations = iter;
            rep->total_spmvms = static_cast<double>(iter) * rep->n_search * rep->degree;
            if (history) {
                double* h = history + 5 * (iter - 1);
                h[0] = iter;
                h[1] = rmin;
                h[2] = rmax;
                h[3] = acc;
                h[4] = rep->total_spmvms;
            }
            rep->n_values = static_cast<int>(nb);
            if (nb > cap) fail(CHEBFD_ERR_INVALID_ARGUMENT, "solve: value capacity too small");
            for (int64_t k = 0; k < nb; ++k) {
                values[k] = ritz.values[k];
                residual_norms[k] = ritz.res[k];
                accepted[k] = acc_flags[k];
            }
            if (pending == 0 && acc >= required) {
                rep->converged = 1;
                break;
            }
            // block restart from the current Ritz vectors; same width: copy into x so the
            // captured filter graph (keyed on x's storage) replays instead of recapturing
            if (ritz.vectors->width == x->width) {
                CFD_CUDA(cudaMemcpyAsync(x->owned(), ritz.vectors->owned(), x->owned_bytes(),
                                         cudaMemcpyDeviceToDevice, c.stream));
            } else {
                x = std::move(ritz.vectors);
                ritz.vectors.reset();
            }
        }
        if (vectors) {
            if (ritz.vectors)
                *vectors = reinterpret_cast<chebfd_block*>(ritz.vectors.release());
            else
                *vectors = reinterpret_cast<chebfd_block*>(x.release());
        }
        rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

}  // extern "C"
