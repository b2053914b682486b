// extern "C" shim over the UNMODIFIED reference library -- TEST INFRASTRUCTURE.
//
// Compiled by oracle/Makefile against /root/reference/proj/include together
// with the reference's own src/*.cpp into oracle/_ref/libchebfd_ref.so.  It
// is the "real reference" leg of the oracle: tests/golden/make_golden.py uses
// it to write golden fixtures, tests use it (when built) to pin the C
// restatement in oracle/chebfd_oracle.c, and bench.py --impl reference times
// it on the host cores.  Nothing in the product library links or loads it.
//
// Every entry point returns 0 on success or a nonzero code naming the C++
// exception type the reference threw (1 invalid_argument, 2 runtime_error,
// 3 domain_error, 4 out_of_range, 9 other); ref_last_error() gives the text.
#include <chebfd/bench.hpp>
#include <chebfd/filter.hpp>
#include <chebfd/filter_design.hpp>
#include <chebfd/kernels.hpp>
#include <chebfd/matrix_market.hpp>
#include <chebfd/models.hpp>
#include <chebfd/parallel.hpp>
#include <chebfd/solver.hpp>
#include <chebfd/spectral.hpp>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

using namespace chebfd;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 4;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

struct RefMatrix {
    int kind = 0;  // 0 real64, 1 complex128
    SparseMatrix<double> r;
    SparseMatrix<Complex> c;
};

Boundary boundary_of(int b) {
    switch (b) {
        case 0: return Boundary::periodic_xy_open_z;
        case 1: return Boundary::periodic_all;
        case 2: return Boundary::open_all;
    }
    throw std::invalid_argument("bad boundary code");
}

Kernel kernel_of(int kind, int mu) {
    switch (kind) {
        case 0: return {KernelKind::None, 0};
        case 1: return {KernelKind::Fejer, 0};
        case 2: return {KernelKind::Jackson, 0};
        case 3: return {KernelKind::Lanczos, mu};
    }
    throw std::invalid_argument("bad kernel code");
}

template <class S>
BlockVector<S> block_in(const void* p, int64_t dim, int64_t width) {
    BlockVector<S> b(dim, width);
    if (dim * width) std::memcpy(b.data(), p, sizeof(S) * static_cast<size_t>(dim * width));
    return b;
}

template <class S>
void block_out(const BlockVector<S>& b, void* p) {
    if (b.size()) std::memcpy(p, b.data(), sizeof(S) * b.size());
}

FilterPolynomial filter_from(const double* combined, int degree, double alpha, double beta) {
    FilterPolynomial p;
    p.degree = degree;
    p.combined.assign(combined, combined + degree + 1);
    p.alpha = alpha;
    p.beta = beta;
    return p;
}

// dispatch on the matrix kind
template <class F>
void with_matrix(void* h, F&& f) {
    auto* m = static_cast<RefMatrix*>(h);
    if (m->kind == 0)
        f(m->r);
    else
        f(m->c);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { set_num_threads(n); }
int ref_num_threads() { return num_threads(); }

// ---- matrices (models.cpp, sparse_matrix.hpp) ----
int ref_graphene(int64_t lx, int64_t ly, double t, double disorder, int boundary, uint64_t seed,
                 void** out) {
    return guard([&] {
        LatticeSpec s;
        s.lx = lx;
        s.ly = ly;
        s.t = t;
        s.disorder = disorder;
        s.boundary = boundary_of(boundary);
        s.seed = seed;
        auto m = std::make_unique<RefMatrix>();
        m->kind = 0;
        m->r = graphene(s);
        *out = m.release();
    });
}

int ref_topological_insulator(int64_t lx, int64_t ly, int64_t lz, double t, double disorder,
                              int boundary, uint64_t seed, void** out) {
    return guard([&] {
        LatticeSpec s;
        s.lx = lx;
        s.ly = ly;
        s.lz = lz;
        s.t = t;
        s.disorder = disorder;
        s.boundary = boundary_of(boundary);
        s.seed = seed;
        auto m = std::make_unique<RefMatrix>();
        m->kind = 1;
        m->c = topological_insulator(s);
        *out = m.release();
    });
}

int ref_diag_flat(int64_t dim, double lo, double hi, void** out) {
    return guard([&] {
        auto m = std::make_unique<RefMatrix>();
        m->r = diag_flat(dim, {lo, hi});
        *out = m.release();
    });
}

int ref_diag_linear(int64_t dim, void** out) {
    return guard([&] {
        auto m = std::make_unique<RefMatrix>();
        m->r = diag_linear(dim);
        *out = m.release();
    });
}

int ref_matrix_from_csr(int kind, int64_t dim, const int64_t* offs, const int64_t* cols,
                        const void* vals, void** out) {
    return guard([&] {
        const int64_t nnz = offs[dim];
        auto m = std::make_unique<RefMatrix>();
        m->kind = kind;
        std::vector<Index> o(offs, offs + dim + 1), c(cols, cols + nnz);
        if (kind == 0) {
            const double* v = static_cast<const double*>(vals);
            m->r = SparseMatrix<double>(dim, std::move(o), std::move(c),
                                        std::vector<double>(v, v + nnz));
        } else {
            const Complex* v = static_cast<const Complex*>(vals);
            m->c = SparseMatrix<Complex>(dim, std::move(o), std::move(c),
                                         std::vector<Complex>(v, v + nnz));
        }
        *out = m.release();
    });
}

void ref_matrix_free(void* h) { delete static_cast<RefMatrix*>(h); }

int ref_matrix_info(void* h, int* kind, int64_t* dim, int64_t* nnz) {
    return guard([&] {
        auto* m = static_cast<RefMatrix*>(h);
        *kind = m->kind;
        with_matrix(h, [&](const auto& a) {
            *dim = a.dim();
            *nnz = a.nnz();
        });
    });
}

int ref_matrix_csr(void* h, int64_t* offs, int64_t* cols, void* vals) {
    return guard([&] {
        with_matrix(h, [&](const auto& a) {
            std::memcpy(offs, a.row_offsets().data(), sizeof(int64_t) * (a.dim() + 1));
            std::memcpy(cols, a.col_indices().data(), sizeof(int64_t) * a.nnz());
            std::memcpy(vals, a.values().data(), sizeof(a.values()[0]) * a.nnz());
        });
    });
}

int ref_matrix_is_hermitian(void* h, double tol, int* out) {
    return guard([&] { with_matrix(h, [&](const auto& a) { *out = a.is_hermitian(tol); }); });
}

// ---- block vectors (block_vector.hpp) ----
int ref_randomize(int kind, int64_t dim, int64_t width, uint64_t seed, void* out) {
    return guard([&] {
        if (kind == 0) {
            BlockVector<double> b(dim, width);
            b.randomize(seed);
            block_out(b, out);
        } else {
            BlockVector<Complex> b(dim, width);
            b.randomize(seed);
            block_out(b, out);
        }
    });
}

// ---- filter coefficients (filter.cpp) ----
int ref_window_coeffs(double tlo, double thi, double blo, double bhi, int degree, double* out) {
    return guard([&] {
        auto c = window_coeffs({tlo, thi}, {blo, bhi}, degree);
        std::memcpy(out, c.data(), sizeof(double) * c.size());
    });
}

int ref_kernel_coeffs(int kind, int mu, int degree, double* out) {
    return guard([&] {
        auto g = kernel_coeffs(kernel_of(kind, mu), degree);
        std::memcpy(out, g.data(), sizeof(double) * g.size());
    });
}

int ref_make_filter(double tlo, double thi, double blo, double bhi, int degree, int kind, int mu,
                    double* combined, double* alpha, double* beta) {
    return guard([&] {
        auto p = make_filter({tlo, thi}, {blo, bhi}, degree, kernel_of(kind, mu));
        std::memcpy(combined, p.combined.data(), sizeof(double) * p.combined.size());
        *alpha = p.alpha;
        *beta = p.beta;
    });
}

int ref_eval_scalar(const double* combined, int degree, double alpha, double beta, double blo,
                    double bhi, double x, double* out) {
    return guard([&] {
        auto p = filter_from(combined, degree, alpha, beta);
        p.bounds = {blo, bhi};
        *out = eval_scalar(p, x);
    });
}

// ---- kernels (kernels.hpp) ----
int ref_spmmvm(void* h, const void* x, int64_t width, double alpha, double beta, void* y) {
    return guard([&] {
        with_matrix(h, [&](const auto& a) {
            using S = std::decay_t<decltype(a.values()[0])>;
            auto X = block_in<S>(x, a.dim(), width);
            block_out(spmmvm(a, X, alpha, beta), y);
        });
    });
}

int ref_spmmvm_fused(void* h, const void* u, void* w, void* x, int64_t width, double alpha,
                     double beta, double coeff, void* dots) {
    return guard([&] {
        with_matrix(h, [&](const auto& a) {
            using S = std::decay_t<decltype(a.values()[0])>;
            auto U = block_in<S>(u, a.dim(), width);
            auto W = block_in<S>(w, a.dim(), width);
            auto X = block_in<S>(x, a.dim(), width);
            spmmvm_fused(a, U, W, X, alpha, beta, coeff, static_cast<S*>(dots));
            block_out(W, w);
            block_out(X, x);
        });
    });
}

int ref_recurrence_step(void* h, const void* u, void* w, int64_t width, double alpha, double beta) {
    return guard([&] {
        with_matrix(h, [&](const auto& a) {
            using S = std::decay_t<decltype(a.values()[0])>;
            auto U = block_in<S>(u, a.dim(), width);
            auto W = block_in<S>(w, a.dim(), width);
            recurrence_step(a, U, W, alpha, beta);
            block_out(W, w);
        });
    });
}

int ref_block_axpy_scal(int kind, int64_t dim, int64_t width, void* x, const void* u,
                        const void* w, double c0, double c1, double c2) {
    return guard([&] {
        auto run = [&](auto tag) {
            using S = decltype(tag);
            auto X = block_in<S>(x, dim, width);
            auto U = block_in<S>(u, dim, width);
            auto W = block_in<S>(w, dim, width);
            block_axpy_scal(X, U, W, c0, c1, c2);
            block_out(X, x);
        };
        kind == 0 ? run(double{}) : run(Complex{});
    });
}

int ref_gram(int kind, int64_t dim, const void* x, int64_t nx, const void* y, int64_t ny,
             void* g) {
    return guard([&] {
        auto run = [&](auto tag) {
            using S = decltype(tag);
            auto G = gram(block_in<S>(x, dim, nx), block_in<S>(y, dim, ny));
            std::memcpy(g, G.a.data(), sizeof(S) * G.a.size());
        };
        kind == 0 ? run(double{}) : run(Complex{});
    });
}

int ref_column_dots(int kind, int64_t dim, int64_t width, const void* x, const void* y, void* d) {
    return guard([&] {
        auto run = [&](auto tag) {
            using S = decltype(tag);
            auto v = column_dots(block_in<S>(x, dim, width), block_in<S>(y, dim, width));
            std::memcpy(d, v.data(), sizeof(S) * v.size());
        };
        kind == 0 ? run(double{}) : run(Complex{});
    });
}

int ref_column_norms(int kind, int64_t dim, int64_t width, const void* x, double* out) {
    return guard([&] {
        auto run = [&](auto tag) {
            using S = decltype(tag);
            auto v = column_norms(block_in<S>(x, dim, width));
            std::memcpy(out, v.data(), sizeof(double) * v.size());
        };
        kind == 0 ? run(double{}) : run(Complex{});
    });
}

int ref_block_mult_small(int kind, int64_t dim, int64_t width, const void* x, const void* b,
                         int64_t bcols, void* y) {
    return guard([&] {
        auto run = [&](auto tag) {
            using S = decltype(tag);
            DenseMatrix<S> B(width, bcols);
            std::memcpy(B.a.data(), b, sizeof(S) * B.a.size());
            block_out(block_mult_small(block_in<S>(x, dim, width), B), y);
        };
        kind == 0 ? run(double{}) : run(Complex{});
    });
}

// ---- filter application (filter.hpp:73-116) ----
int ref_apply_filter(void* h, void* x, int64_t width, const double* combined, int degree,
                     double alpha, double beta, double* moments) {
    return guard([&] {
        with_matrix(h, [&](const auto& a) {
            using S = std::decay_t<decltype(a.values()[0])>;
            auto X = block_in<S>(x, a.dim(), width);
            auto p = filter_from(combined, degree, alpha, beta);
            auto m = apply_filter(a, X, p, moments != nullptr);
            block_out(X, x);
            if (moments && m) std::memcpy(moments, m->m.data(), sizeof(double) * m->m.size());
        });
    });
}

// Time k fused steps (filter.hpp:107-114 inner loop) on fresh blocks; used by
// bench.py --impl reference as a bounded sample of apply_filter.
int ref_time_fused_steps(void* h, int64_t width, int steps, double alpha, double beta,
                         double coeff, uint64_t seed, double* seconds) {
    return guard([&] {
        with_matrix(h, [&](const auto& a) {
            using S = std::decay_t<decltype(a.values()[0])>;
            BlockVector<S> u(a.dim(), width), w(a.dim(), width), x(a.dim(), width);
            u.randomize(seed);
            w.randomize(seed + 1);
            x.randomize(seed + 2);
            BlockVector<S>* pu = &u;
            BlockVector<S>* pw = &w;
            spmmvm_fused(a, *pu, *pw, x, alpha, beta, coeff);  // warm-up (page faults)
            const auto t0 = std::chrono::steady_clock::now();
            for (int n = 0; n < steps; ++n) {
                std::swap(pu, pw);
                spmmvm_fused(a, *pu, *pw, x, alpha, beta, coeff);
            }
            *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        });
    });
}

// A persistent steady-state timing session for the CPU baseline: U, W, X blocks of the
// reference's own BlockVector type allocated and filled once (a cheap deterministic
// fill, touched in parallel so the pages are resident), then repeated calls timing
// `steps` reference spmmvm_fused steps (kernels.hpp:74-118) with pointer swaps as
// apply_filter's loop does (filter.hpp:105-114).  Timing infrastructure, not a kernel.
struct FusedSession {
    void* h = nullptr;
    int64_t width = 0;
    BlockVector<double> ru, rw, rx;
    BlockVector<Complex> cu, cw, cx;
};

int ref_fused_session_create(void* h, int64_t width, void** out) {
    return guard([&] {
        auto s = std::make_unique<FusedSession>();
        s->h = h;
        s->width = width;
        with_matrix(h, [&](const auto& a) {
            using S = std::decay_t<decltype(a.values()[0])>;
            auto fill = [&](BlockVector<S>& b, double phase) {
                b = BlockVector<S>(a.dim(), width);
                S* d = b.data();
                const int64_t n = a.dim() * width;
#pragma omp parallel for schedule(static)
                for (int64_t i = 0; i < n; ++i) {
                    const double v = std::sin(0.001 * static_cast<double>(i % 100003) + phase);
                    if constexpr (std::is_same_v<S, Complex>)
                        d[i] = Complex(v, 0.5 * v);
                    else
                        d[i] = v;
                }
            };
            if constexpr (std::is_same_v<S, Complex>) {
                fill(s->cu, 0.1);
                fill(s->cw, 0.2);
                fill(s->cx, 0.3);
            } else {
                fill(s->ru, 0.1);
                fill(s->rw, 0.2);
                fill(s->rx, 0.3);
            }
        });
        *out = s.release();
    });
}

int ref_fused_session_run(void* sess, int steps, double alpha, double beta, double coeff,
                          double* seconds) {
    return guard([&] {
        auto* s = static_cast<FusedSession*>(sess);
        with_matrix(s->h, [&](const auto& a) {
            using S = std::decay_t<decltype(a.values()[0])>;
            BlockVector<S>*pu, *pw, *px;
            if constexpr (std::is_same_v<S, Complex>) {
                pu = &s->cu; pw = &s->cw; px = &s->cx;
            } else {
                pu = &s->ru; pw = &s->rw; px = &s->rx;
            }
            const auto t0 = std::chrono::steady_clock::now();
            for (int n = 0; n < steps; ++n) {
                spmmvm_fused(a, *pu, *pw, *px, alpha, beta, coeff);
                std::swap(pu, pw);
            }
            *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if constexpr (std::is_same_v<S, Complex>) {
                if (pu != &s->cu) std::swap(s->cu, s->cw);
            } else {
                if (pu != &s->ru) std::swap(s->ru, s->rw);
            }
        });
    });
}

// the reference's apply_filter (filter.hpp:73-116) on the session's X block, in place,
// timed around the call alone (its own start-up allocations included)
int ref_fused_session_apply(void* sess, const double* combined, int degree, double alpha,
                            double beta, double* seconds) {
    return guard([&] {
        auto* s = static_cast<FusedSession*>(sess);
        with_matrix(s->h, [&](const auto& a) {
            using S = std::decay_t<decltype(a.values()[0])>;
            BlockVector<S>* px;
            if constexpr (std::is_same_v<S, Complex>)
                px = &s->cx;
            else
                px = &s->rx;
            auto p = filter_from(combined, degree, alpha, beta);
            const auto t0 = std::chrono::steady_clock::now();
            auto m = apply_filter(a, *px, p, false);
            *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            (void)m;
        });
    });
}

// the reference's gram(X, X) (kernels.hpp:165-192) of the session's X block, timed
int ref_fused_session_gram(void* sess, double* seconds) {
    return guard([&] {
        auto* s = static_cast<FusedSession*>(sess);
        with_matrix(s->h, [&](const auto& a) {
            using S = std::decay_t<decltype(a.values()[0])>;
            const auto t0 = std::chrono::steady_clock::now();
            if constexpr (std::is_same_v<S, Complex>) {
                auto g = gram(s->cx, s->cx);
                (void)g;
            } else {
                auto g = gram(s->rx, s->rx);
                (void)g;
            }
            *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        });
    });
}

void ref_fused_session_free(void* sess) { delete static_cast<FusedSession*>(sess); }

// ---- solver pieces (solver.cpp) ----
int ref_svqb(int kind, int64_t dim, int64_t width, const void* y, double drop_tol, void* q,
             int64_t* rank) {
    return guard([&] {
        auto run = [&](auto tag) {
            using S = decltype(tag);
            auto r = svqb_orthonormalize(block_in<S>(y, dim, width), drop_tol);
            *rank = r.rank;
            block_out(r.q, q);
        };
        kind == 0 ? run(double{}) : run(Complex{});
    });
}

int ref_rayleigh_ritz(void* h, const void* q, int64_t width, void* v, double* values,
                      double* resnorms) {
    return guard([&] {
        with_matrix(h, [&](const auto& a) {
            using S = std::decay_t<decltype(a.values()[0])>;
            auto r = rayleigh_ritz(a, block_in<S>(q, a.dim(), width));
            block_out(r.vectors, v);
            std::memcpy(values, r.values.data(), sizeof(double) * r.values.size());
            std::memcpy(resnorms, r.residual_norms.data(), sizeof(double) * r.values.size());
        });
    });
}

// ---- spectral probes (spectral.cpp) ----
int ref_lanczos_bounds(void* h, int iters, uint64_t seed, double* lo, double* hi) {
    return guard([&] {
        with_matrix(h, [&](const auto& a) {
            auto b = lanczos_bounds(a, iters, seed);
            *lo = b.lo;
            *hi = b.hi;
        });
    });
}

int ref_kpm_dos(void* h, double blo, double bhi, int order, int samples, uint64_t seed,
                double* mu) {
    return guard([&] {
        with_matrix(h, [&](const auto& a) {
            auto d = kpm_dos(a, {blo, bhi}, order, samples, seed);
            std::memcpy(mu, d.moments().data(), sizeof(double) * d.moments().size());
        });
    });
}

int ref_dos_count(const double* mu, int order, double blo, double bhi, double lo, double hi,
                  double* out) {
    return guard([&] {
        DosEstimate d(std::vector<double>(mu, mu + order + 1), {blo, bhi}, 1, 1);
        *out = d.count(lo, hi);
    });
}

int ref_choose_parameters(const double* mu, int order, double blo, double bhi, double tlo,
                          double thi, double n_search, int kkind, int mu_k, double epsilon,
                          int* np_opt, double* sigma, double* eta, double* delta_prime) {
    return guard([&] {
        DosEstimate d(std::vector<double>(mu, mu + order + 1), {blo, bhi}, 1, 1);
        auto cp = choose_parameters(d, {tlo, thi}, n_search, kernel_of(kkind, mu_k), epsilon);
        *np_opt = cp.design.np_opt;
        *sigma = cp.design.sigma;
        *eta = cp.design.eta_opt;
        *delta_prime = cp.cfg.delta_prime;
    });
}

struct RefSolveOptions {
    double target_lo, target_hi;
    double epsilon;
    int n_search;
    int degree;
    int kernel_kind, kernel_mu;
    int max_iters;
    uint64_t seed;
    int dos_moments, dos_samples;
    double bounds_lo, bounds_hi;
    int collect_weight_density;
};

struct RefSolveReport {
    int converged, iterations, n_search, degree, n_values;
    double total_spmvms, sigma, eta, bounds_lo, bounds_hi, matrix_norm_est, n_target_estimate;
    double seconds;
    double weight_integral;
};

// values/resnorms/accepted need capacity >= n_search (max_values); history
// holds (iter, rmin, rmax, accepted, spmvms) x max_iters.
int ref_solve(void* h, const RefSolveOptions* o, RefSolveReport* rep, int max_values,
              double* values, double* resnorms, int* accepted, double* history) {
    return guard([&] {
        SolverOptions opts;
        opts.target = {o->target_lo, o->target_hi};
        opts.epsilon = o->epsilon;
        opts.n_search = o->n_search;
        opts.degree = o->degree;
        opts.kernel = kernel_of(o->kernel_kind, o->kernel_mu);
        opts.max_iters = o->max_iters;
        opts.seed = o->seed;
        opts.dos_moments = o->dos_moments;
        opts.dos_samples = o->dos_samples;
        opts.bounds = {o->bounds_lo, o->bounds_hi};
        opts.collect_weight_density = o->collect_weight_density != 0;
        with_matrix(h, [&](const auto& a) {
            auto r = solve(a, opts);
            rep->converged = r.converged;
            rep->iterations = r.iterations;
            rep->n_search = r.n_search;
            rep->degree = r.degree;
            rep->total_spmvms = r.total_spmvms;
            rep->sigma = r.sigma;
            rep->eta = r.eta;
            rep->bounds_lo = r.bounds.lo;
            rep->bounds_hi = r.bounds.hi;
            rep->matrix_norm_est = r.matrix_norm_est;
            rep->n_target_estimate = r.n_target_estimate;
            rep->seconds = r.seconds;
            rep->weight_integral = r.have_weight ? r.weight.integral() : 0.0;
            const int n = static_cast<int>(r.ritz.values.size());
            rep->n_values = n;
            if (n > max_values) throw std::invalid_argument("ref_solve: value capacity too small");
            for (int k = 0; k < n; ++k) {
                values[k] = r.ritz.values[k];
                resnorms[k] = r.ritz.residual_norms[k];
                accepted[k] = r.ritz.accepted[k] ? 1 : 0;
            }
            if (history)
                for (size_t i = 0; i < r.history.size() && static_cast<int>(i) < o->max_iters;
                     ++i) {
                    history[5 * i + 0] = r.history[i].iteration;
                    history[5 * i + 1] = r.history[i].min_residual;
                    history[5 * i + 2] = r.history[i].max_residual;
                    history[5 * i + 3] = r.history[i].accepted_count;
                    history[5 * i + 4] = r.history[i].cumulative_spmvms;
                }
        });
    });
}

// ---- bench conventions (bench.cpp:28-42) ----
int ref_intensity_model(double n_nzr, int s_d, int s_i, int f_a, int f_m, int n_b, double* out) {
    return guard([&] {
        IntensityParams p{n_nzr, s_d, s_i, f_a, f_m};
        *out = intensity_model(p, n_b);
    });
}

// ---- on-disk formats (matrix_market.cpp, block_vector.hpp:63-96) ----
int ref_read_matrix_market(const char* path, void** out, int* hermitian) {
    return guard([&] {
        MatrixVariant v = read_matrix_market(path);
        auto m = std::make_unique<RefMatrix>();
        if (std::holds_alternative<SparseMatrix<double>>(v)) {
            m->kind = 0;
            m->r = std::get<SparseMatrix<double>>(std::move(v));
            *hermitian = m->r.hermitian_flag();
        } else {
            m->kind = 1;
            m->c = std::get<SparseMatrix<Complex>>(std::move(v));
            *hermitian = m->c.hermitian_flag();
        }
        *out = m.release();
    });
}

int ref_write_matrix_market(void* h, const char* path, int hermitian) {
    return guard([&] {
        with_matrix(h, [&](const auto& a) {
            using M = std::decay_t<decltype(a)>;
            M flagged(a.dim(), a.row_offsets(), a.col_indices(), a.values(), hermitian != 0);
            write_matrix_market(path, flagged);
        });
    });
}

int ref_block_save(int kind, int64_t dim, int64_t width, const void* data, const char* path) {
    return guard([&] {
        if (kind == 0)
            block_in<double>(data, dim, width).save(path);
        else
            block_in<Complex>(data, dim, width).save(path);
    });
}

// loads as scalar kind `kind` (BlockVector<S>::load); data == nullptr: shape only
int ref_block_load(int kind, const char* path, int64_t* dim, int64_t* width, void* data) {
    return guard([&] {
        auto take = [&](const auto& b) {
            *dim = b.dim();
            *width = b.width();
            if (data) block_out(b, data);
        };
        if (kind == 0)
            take(BlockVector<double>::load(path));
        else
            take(BlockVector<Complex>::load(path));
    });
}

// ---- bench front end (bench.cpp:71-126); out[8 * k] = n_b, seconds, flops, gflops,
// gbs_proxy, intensity, roofline, efficiency of point k
int ref_bench_filter(void* h, const int* sizes, int n, int degree, double bandwidth, double* out) {
    return guard([&] {
        with_matrix(h, [&](const auto& a) {
            const BenchReport rep =
                bench_filter(a, std::vector<int>(sizes, sizes + n), degree, bandwidth);
            for (size_t k = 0; k < rep.points.size(); ++k) {
                const BenchPoint& p = rep.points[k];
                const double row[8] = {double(p.n_b), p.seconds,   p.flops,     p.gflops,
                                       p.gbs_proxy,   p.intensity, p.roofline, p.efficiency};
                std::memcpy(out + 8 * k, row, sizeof row);
            }
        });
    });
}

// damping_factor (filter_design.cpp:178-184) of make_filter(target, bounds, degree, kernel)
int ref_damping_factor(double tlo, double thi, double dprime, double blo, double bhi, int degree,
                       int kind, int mu, double* out) {
    return guard([&] {
        const FilterPolynomial p = make_filter({tlo, thi}, {blo, bhi}, degree, kernel_of(kind, mu));
        IntervalConfig cfg;
        cfg.target = {tlo, thi};
        cfg.delta_prime = dprime;
        cfg.bounds = {blo, bhi};
        *out = damping_factor(p, cfg);
    });
}

}  // extern "C"
