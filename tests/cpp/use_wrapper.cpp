// Example / test of the C++ drop-in layer (include/chebfd_b200.hpp).
//   use_wrapper --host-only   host-side pieces only (no GPU needed)
//   use_wrapper               full device path (needs a B200)
// Exit code 0 on success.
#include <chebfd_b200.hpp>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>

namespace cb = chebfd::b200;

static int fails = 0;
#define EXPECT(c)                                                       \
    do {                                                                \
        if (!(c)) {                                                     \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);     \
            ++fails;                                                    \
        }                                                               \
    } while (0)

int main(int argc, char** argv) {
    const bool host_only = argc > 1 && std::strcmp(argv[1], "--host-only") == 0;
    // test_filter.cpp:34-39 closed forms
    auto c = cb::window_coeffs({-0.5, 0.5}, {-1.0, 1.0}, 4);
    EXPECT(std::abs(c[0] - 1.0 / 3.0) < 1e-14);
    EXPECT(std::abs(c[2] + std::sqrt(3.0) / M_PI) < 1e-14);
    auto p = cb::make_filter({-0.2, 0.3}, {-1.0, 1.0}, 40, {cb::KernelKind::Lanczos, 2});
    EXPECT(p.combined.size() == 41);
    bool threw = false;
    try {
        cb::eval_scalar(p, 1.5);
    } catch (const std::domain_error&) {
        threw = true;
    }
    EXPECT(threw);
    threw = false;
    try {
        cb::make_filter({0.3, -0.2}, {-1.0, 1.0}, 40, {});
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw);
    // Matrix Market writer (host): 2x2 symmetric, lower triangle only
    const std::string dir = argc > 2 ? argv[2] : ".";
    const std::string mtx = dir + "/use_wrapper.mtx";
    cb::write_matrix_market<double>(mtx, 2, {0, 2, 4}, {0, 1, 0, 1}, {2.0, -1.0, -1.0, 2.0});
    if (std::FILE* f = std::fopen(mtx.c_str(), "r")) {
        char buf[256] = {0};
        const size_t got = std::fread(buf, 1, sizeof buf - 1, f);
        std::fclose(f);
        EXPECT(got > 0 && std::strcmp(buf, "%%MatrixMarket matrix coordinate real symmetric\n"
                                           "2 2 3\n1 1 2\n2 1 -1\n2 2 2\n") == 0);
    } else {
        EXPECT(false);
    }
    if (host_only) {
        threw = false;
        try {
            cb::Context ctx(0);
        } catch (const cb::CudaError&) {
            threw = true;  // no GPU here: fail loudly, no CPU fallback
        }
        EXPECT(threw);
        std::printf("%s (host-only)\n", fails ? "FAILED" : "ok");
        return fails;
    }
    cb::Context ctx(0);
    cb::LatticeSpec spec;
    spec.lx = spec.ly = spec.lz = 6;
    spec.disorder = 0.5;
    auto A = cb::topological_insulator(ctx, spec);
    EXPECT(A.dim() == 4 * 216);
    cb::BlockVector<cb::Complex> X(A, 8);
    X.randomize(3);
    auto pf = cb::make_filter({-0.3, 0.3}, {-5.6, 5.6}, 40, {cb::KernelKind::Lanczos, 2});
    auto m = cb::apply_filter(A, X, pf, true);
    EXPECT(m.has_value() && m->degree == 40);
    auto n = cb::column_norms(X);
    EXPECT(n.size() == 8 && std::isfinite(n[0]) && n[0] > 0);
    auto G = cb::gram(X, X);
    EXPECT(std::abs(G(0, 0).real() - n[0] * n[0]) < 1e-10 * n[0] * n[0]);
    threw = false;
    try {
        cb::spmmvm_fused(A, X, X, X, 1.0, 0.0, 0.5);
    } catch (const std::invalid_argument&) {
        threw = true;  // test_core_linalg.cpp:157-164
    }
    EXPECT(threw);
    // file round trips on the device path
    auto V = cb::read_matrix_market(ctx, mtx);
    EXPECT(V.index() == 0 && std::get<0>(V).dim() == 2 && std::get<0>(V).nnz() == 4);
    X.save(dir + "/use_wrapper.cbfd");
    auto Y = cb::BlockVector<cb::Complex>::load(A, dir + "/use_wrapper.cbfd");
    EXPECT(Y.download() == X.download());
    // a stream of host blocks through FilterPipe = apply_filter_host, bit for bit
    std::vector<cb::Complex> h1 = Y.download(), h2 = h1, h3 = h1, h4(h1.size());
    cb::apply_filter_host(A, h1, 8, pf);
    {
        cb::FilterPipe<cb::Complex> pipe(A, 8);
        pipe.submit(h2.data(), h2.data(), pf);
        pipe.submit(h3.data(), h4.data(), pf);
        pipe.wait();
    }
    EXPECT(h1 == h2 && h1 == h4);
    // moments by direct <x0, w> dots vs the doubling identities: same table to rounding
    cb::BlockVector<cb::Complex> Z(A, 8);
    Z.randomize(3);
    ctx.set_option(CHEBFD_OPT_MOMENTS, 0);
    auto md = cb::apply_filter(A, Z, pf, true);
    ctx.set_option(CHEBFD_OPT_MOMENTS, 1);
    double worst = 0.0;
    for (size_t i = 0; i < md->m.size(); ++i) worst = std::max(worst, std::abs(md->m[i] - m->m[i]));
    EXPECT(worst <= 1e-12 * std::abs(m->m[0]));
    // block_mult_small(X, B) (kernels.hpp:216-232): X times the identity is X
    cb::DenseMatrix<cb::Complex> I(8, 3);
    for (int k = 0; k < 3; ++k) I(k, k) = 1.0;
    auto X3 = cb::block_mult_small(X, I);
    EXPECT(X3.width() == 3 && X3.dim() == X.dim());
    {
        auto a = X.download(), b = X3.download();
        bool same = true;
        for (cb::Index i = 0; i < X.dim(); ++i)
            for (int k = 0; k < 3; ++k) same = same && a[i * 8 + k] == b[i * 3 + k];
        EXPECT(same);
    }
    // svqb_orthonormalize + rayleigh_ritz (solver.cpp:32-91): orthonormal Q, ascending
    // values with residuals; a duplicated column drops the rank by one
    auto sq = cb::svqb_orthonormalize(X);
    EXPECT(sq.rank == 8 && sq.q.width() == 8);
    auto Gq = cb::gram(sq.q, sq.q);
    double off = 0.0;
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) off = std::max(off, std::abs(Gq(i, j) - (i == j ? 1.0 : 0.0)));
    EXPECT(off < 1e-12);
    cb::DenseMatrix<cb::Complex> dup(8, 8);
    for (int k = 0; k < 8; ++k) dup(k, k) = 1.0;
    dup(0, 7) = 1.0;
    dup(7, 7) = 0.0;  // column 7 := column 0
    auto Xd = cb::block_mult_small(X, dup);
    auto sd = cb::svqb_orthonormalize(Xd);
    EXPECT(sd.rank == 7 && sd.q.width() == 7);
    auto rz = cb::rayleigh_ritz(A, sq.q);
    EXPECT(rz.values.size() == 8 && rz.vectors.width() == 8 && rz.residual_norms.size() == 8);
    EXPECT(std::is_sorted(rz.values.begin(), rz.values.end()));
    // spectral.hpp: kpm_dos + estimate_count (interval outside the bounds throws)
    auto bnd = cb::lanczos_bounds(A, 30, 1);
    auto dos = cb::kpm_dos(A, bnd, 200, 8, 2);
    EXPECT(dos.moments().size() == 201 && dos.num_samples() == 8 && dos.matrix_dim() == A.dim());
    const double all = cb::estimate_count(dos, bnd);
    EXPECT(std::abs(all - double(A.dim())) < 0.05 * double(A.dim()));
    EXPECT(dos.density(0.5 * (bnd.lo + bnd.hi)) >= 0.0);
    threw = false;
    try {
        cb::estimate_count(dos, {bnd.lo - 1.0, bnd.hi});
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw);
    // weight_density of the filter moments integrates to the summed squared column norms
    auto wd = cb::weight_density(*m, pf.bounds);
    double m0 = 0.0;
    for (int k = 0; k < 8; ++k) m0 += (*m)(0, k);
    EXPECT(wd.integral() == m0 && wd.moments().size() == 41);
    // solve (solver.cpp:93-214) on a tiny window: the report carries the Ritz set, the
    // history and the weight density of the last filter (solver.cpp:158-162)
    cb::SolverOptions so;
    so.target = {-0.3, 0.3};
    so.n_search = 16;
    so.degree = 60;
    auto rep = cb::solve(A, so);
    EXPECT(rep.iterations >= 1 && static_cast<int>(rep.history.size()) == rep.iterations);
    EXPECT(rep.have_weight && static_cast<int>(rep.weight.moments().size()) == rep.degree + 1);
    EXPECT(std::abs(rep.weight.integral() - 16.0) < 1e-9);
    EXPECT(rep.ritz.vectors.width() == static_cast<cb::Index>(rep.ritz.values.size()));
    std::printf("%s (device)\n", fails ? "FAILED" : "ok");
    return fails;
}
