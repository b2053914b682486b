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
    std::printf("%s (device)\n", fails ? "FAILED" : "ok");
    return fails;
}
