// chebfd_b200.hpp -- the reference's C++ driver API, backed by the sm_100a
// library through the C ABI in chebfd_b200.h.
//
// A caller of /root/reference/proj/include/chebfd/*.hpp switches by
// replacing `chebfd::` with `chebfd::b200::` and passing a Context: the
// template signatures (double / std::complex<double>), argument meaning,
// return types and exception types (std::invalid_argument,
// std::runtime_error, std::domain_error, std::out_of_range) are the
// reference's.  Sparse matrices and block vectors live on the GPU; upload /
// download move row-major host data (block_vector.hpp:15-16).
#pragma once

#include <complex>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <variant>
#include <vector>

#include "chebfd_b200.h"

namespace chebfd::b200 {

using Index = std::int64_t;
using Complex = std::complex<double>;

template <class S>
inline constexpr int kind_of = std::is_same_v<S, Complex> ? CHEBFD_COMPLEX128 : CHEBFD_REAL64;

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == CHEBFD_OK) return;
    const std::string m = chebfd_last_error();
    switch (rc) {
        case CHEBFD_ERR_INVALID_ARGUMENT: throw std::invalid_argument(m);
        case CHEBFD_ERR_DOMAIN: throw std::domain_error(m);
        case CHEBFD_ERR_OUT_OF_RANGE: throw std::out_of_range(m);
        case CHEBFD_ERR_CUDA:
        case CHEBFD_ERR_NCCL: throw CudaError(m);
        default: throw std::runtime_error(m);
    }
}

// ---- context (replaces the OpenMP runtime, parallel.hpp) ---------------------------
class Context {
  public:
    explicit Context(int device = 0) { check(chebfd_ctx_create(device, &h_)); }
    Context(int device, int rank, int nranks, const unsigned char id[128]) {
        check(chebfd_ctx_create_dist(device, rank, nranks, id, &h_));
    }
    ~Context() {
        if (h_) chebfd_ctx_destroy(h_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    chebfd_ctx* get() const { return h_; }
    void synchronize() { check(chebfd_ctx_synchronize(h_)); }
    // CHEBFD_OPT_* (chebfd_b200.h); drops captured filter graphs
    void set_option(int option, std::int64_t value) { check(chebfd_ctx_set_option(h_, option, value)); }

  private:
    chebfd_ctx* h_ = nullptr;
};

// ---- intervals, kernels, lattice (filter.hpp, models.hpp) ---------------------------
struct Interval {
    double lo = 0.0, hi = 0.0;
    double width() const { return hi - lo; }
    double half_width() const { return 0.5 * (hi - lo); }
    double center() const { return 0.5 * (lo + hi); }
    bool contains(double x) const { return x >= lo && x <= hi; }
    bool contains(const Interval& o) const { return lo <= o.lo && o.hi <= hi; }
};

enum class KernelKind { None = CHEBFD_KERNEL_NONE, Fejer = CHEBFD_KERNEL_FEJER,
                        Jackson = CHEBFD_KERNEL_JACKSON, Lanczos = CHEBFD_KERNEL_LANCZOS };
struct Kernel {
    KernelKind kind = KernelKind::Lanczos;
    int mu = 2;
};

enum class Boundary { periodic_xy_open_z = CHEBFD_PERIODIC_XY_OPEN_Z,
                      periodic_all = CHEBFD_PERIODIC_ALL, open_all = CHEBFD_OPEN_ALL };
struct LatticeSpec {
    Index lx = 1, ly = 1, lz = 1;
    double t = 1.0;
    double disorder = 0.0;
    Boundary boundary = Boundary::periodic_xy_open_z;
    std::uint64_t seed = 1;
    chebfd_lattice c() const {
        return {lx, ly, lz, t, disorder, static_cast<int>(boundary), seed};
    }
};

// ---- device sparse matrix (SELL-C-sigma) -----------------------------------------------
template <class S>
class SparseMatrix {
  public:
    SparseMatrix(Context& ctx, Index dim, const std::vector<Index>& row_offsets,
                 const std::vector<Index>& col_indices, const std::vector<S>& values) {
        if (static_cast<Index>(row_offsets.size()) != dim + 1)
            throw std::invalid_argument("SparseMatrix: row_offsets length must be dim+1");
        if (col_indices.size() != values.size())
            throw std::invalid_argument("SparseMatrix: col/value length mismatch");
        chebfd_matrix* h = nullptr;
        check(chebfd_matrix_from_csr(ctx.get(), kind_of<S>, dim, row_offsets.data(),
                                     col_indices.data(), values.data(), &h));
        h_.reset(h);
    }
    explicit SparseMatrix(chebfd_matrix* h) : h_(h) {}
    Index dim() const { return info().dim; }
    Index nnz() const { return info().nnz; }
    double avg_nonzeros_per_row() const { return dim() ? double(nnz()) / double(dim()) : 0.0; }
    chebfd_matrix_info info() const {
        chebfd_matrix_info i{};
        check(chebfd_matrix_get_info(h_.get(), &i));
        return i;
    }
    chebfd_matrix* get() const { return h_.get(); }

  private:
    struct Del {
        void operator()(chebfd_matrix* m) const { chebfd_matrix_destroy(m); }
    };
    std::unique_ptr<chebfd_matrix, Del> h_;
};

inline SparseMatrix<double> graphene(Context& ctx, const LatticeSpec& s) {
    chebfd_matrix* h = nullptr;
    const chebfd_lattice l = s.c();
    check(chebfd_matrix_graphene(ctx.get(), &l, &h));
    return SparseMatrix<double>(h);
}

inline SparseMatrix<Complex> topological_insulator(Context& ctx, const LatticeSpec& s) {
    chebfd_matrix* h = nullptr;
    const chebfd_lattice l = s.c();
    check(chebfd_matrix_topological_insulator(ctx.get(), &l, &h));
    return SparseMatrix<Complex>(h);
}

// ---- Matrix Market (matrix_market.hpp) ---------------------------------------------------
using MatrixVariant = std::variant<SparseMatrix<double>, SparseMatrix<Complex>>;

// read_matrix_market (matrix_market.cpp:98-115), straight to a device matrix
inline MatrixVariant read_matrix_market(Context& ctx, const std::string& path) {
    chebfd_matrix* h = nullptr;
    check(chebfd_matrix_from_matrix_market(ctx.get(), path.c_str(), &h));
    chebfd_matrix_info i{};
    const int rc = chebfd_matrix_get_info(h, &i);
    if (rc != CHEBFD_OK) {
        chebfd_matrix_destroy(h);
        check(rc);
    }
    if (i.kind == CHEBFD_COMPLEX128) return MatrixVariant(std::in_place_index<1>, h);
    return MatrixVariant(std::in_place_index<0>, h);
}

// write_matrix_market (matrix_market.cpp:63-95) of a host CSR
template <class S>
void write_matrix_market(const std::string& path, Index dim, const std::vector<Index>& row_offsets,
                         const std::vector<Index>& col_indices, const std::vector<S>& values,
                         bool hermitian = true) {
    if (static_cast<Index>(row_offsets.size()) != dim + 1 || col_indices.size() != values.size())
        throw std::invalid_argument("write_matrix_market: inconsistent CSR arrays");
    check(chebfd_write_matrix_market(path.c_str(), kind_of<S>, dim, row_offsets.data(),
                                     col_indices.data(), values.data(), hermitian ? 1 : 0));
}

// ---- device block vector -----------------------------------------------------------------
template <class S>
class BlockVector {
  public:
    BlockVector(const SparseMatrix<S>& a, Index width) {
        chebfd_block* h = nullptr;
        check(chebfd_block_create(a.get(), width, &h));
        h_.reset(h);
    }
    // a zero-filled block with the rows (partition, halos) of `like`, `width` columns
    BlockVector(const BlockVector& like, Index width) {
        chebfd_block* h = nullptr;
        check(chebfd_block_create_like(like.get(), width, &h));
        h_.reset(h);
    }
    BlockVector() = default;  // empty (as the reference's default-constructed BlockVector)
    explicit BlockVector(chebfd_block* h) : h_(h) {}
    BlockVector(BlockVector&&) noexcept = default;
    BlockVector& operator=(BlockVector&&) noexcept = default;
    Index dim() const { return h_ ? info(1) : 0; }
    Index width() const { return h_ ? info(2) : 0; }
    void upload(const std::vector<S>& host) {
        if (static_cast<Index>(host.size()) != dim() * width())
            throw std::invalid_argument("BlockVector::upload: size mismatch");
        check(chebfd_block_upload(h_.get(), host.data()));
    }
    std::vector<S> download() const {
        std::vector<S> out(static_cast<size_t>(dim() * width()));
        check(chebfd_block_download(h_.get(), out.data()));
        return out;
    }
    void randomize(std::uint64_t seed) { check(chebfd_block_randomize(h_.get(), seed)); }
    // BlockVector::save / load (block_vector.hpp:65-95), .cbfd format
    void save(const std::string& path) const { check(chebfd_block_save(h_.get(), path.c_str())); }
    static BlockVector load(const SparseMatrix<S>& a, const std::string& path) {
        chebfd_block* h = nullptr;
        check(chebfd_block_load(a.get(), path.c_str(), &h));
        return BlockVector(h);
    }
    chebfd_block* get() const { return h_.get(); }

  private:
    Index info(int what) const {
        int k = 0;
        int64_t r = 0, w = 0, b = 0;
        check(chebfd_block_info(h_.get(), &k, &r, &w, &b));
        return what == 1 ? r : w;
    }
    struct Del {
        void operator()(chebfd_block* b) const { chebfd_block_destroy(b); }
    };
    std::unique_ptr<chebfd_block, Del> h_;
};

template <class S>
struct DenseMatrix {
    Index rows = 0, cols = 0;
    std::vector<S> a;
    DenseMatrix() = default;
    DenseMatrix(Index r, Index c) : rows(r), cols(c), a(static_cast<size_t>(r * c), S{}) {}
    S& operator()(Index i, Index j) { return a[static_cast<size_t>(i * cols + j)]; }
    const S& operator()(Index i, Index j) const { return a[static_cast<size_t>(i * cols + j)]; }
};

// ---- kernels (kernels.hpp) ------------------------------------------------------------------
template <class S>
BlockVector<S> spmmvm(const SparseMatrix<S>& A, const BlockVector<S>& X, double alpha, double beta) {
    BlockVector<S> Y(A, X.width());
    check(chebfd_spmmvm(A.get(), X.get(), Y.get(), alpha, beta));
    return Y;
}

template <class S>
void spmmvm_fused(const SparseMatrix<S>& A, const BlockVector<S>& U, BlockVector<S>& W,
                  BlockVector<S>& X, double alpha, double beta, double coeff, S* dots = nullptr) {
    check(chebfd_spmmvm_fused(A.get(), U.get(), W.get(), X.get(), alpha, beta, coeff, dots));
}

template <class S>
void recurrence_step(const SparseMatrix<S>& A, const BlockVector<S>& U, BlockVector<S>& W,
                     double alpha, double beta) {
    check(chebfd_recurrence_step(A.get(), U.get(), W.get(), alpha, beta));
}

template <class S>
void block_axpy_scal(BlockVector<S>& X, const BlockVector<S>& U, const BlockVector<S>& W,
                     double c0, double c1, double c2) {
    check(chebfd_block_axpy_scal(X.get(), U.get(), W.get(), c0, c1, c2));
}

template <class S>
DenseMatrix<S> gram(const BlockVector<S>& X, const BlockVector<S>& Y) {
    DenseMatrix<S> G(X.width(), Y.width());
    check(chebfd_gram(X.get(), Y.get(), G.a.data()));
    return G;
}

template <class S>
std::vector<S> column_dots(const BlockVector<S>& X, const BlockVector<S>& Y) {
    std::vector<S> d(static_cast<size_t>(X.width()));
    check(chebfd_column_dots(X.get(), Y.get(), d.data()));
    return d;
}

template <class S>
std::vector<double> column_norms(const BlockVector<S>& X) {
    std::vector<double> n(static_cast<size_t>(X.width()));
    check(chebfd_column_norms(X.get(), n.data()));
    return n;
}

// block_mult_small (kernels.hpp:216-232): Y = X B, B a small n_b x m row-major matrix
template <class S>
BlockVector<S> block_mult_small(const BlockVector<S>& X, const DenseMatrix<S>& B) {
    if (X.width() != B.rows) throw std::invalid_argument("block_mult_small: shape mismatch");
    BlockVector<S> Y(X, B.cols);
    check(chebfd_block_mult_small(X.get(), B.a.data(), B.cols, Y.get()));
    return Y;
}

// ---- filter (filter.hpp) -----------------------------------------------------------------------
struct FilterPolynomial {
    int degree = 0;
    std::vector<double> combined;
    double alpha = 1.0, beta = 0.0;
    Interval target, bounds;
    Kernel kernel;
};

inline std::vector<double> window_coeffs(Interval target, Interval bounds, int degree) {
    std::vector<double> c(static_cast<size_t>(degree < 0 ? 0 : degree) + 1);
    check(chebfd_window_coeffs(target.lo, target.hi, bounds.lo, bounds.hi, degree, c.data()));
    return c;
}

inline std::vector<double> kernel_coeffs(Kernel k, int degree) {
    std::vector<double> g(static_cast<size_t>(degree < 0 ? 0 : degree) + 1);
    check(chebfd_kernel_coeffs(static_cast<int>(k.kind), k.mu, degree, g.data()));
    return g;
}

inline FilterPolynomial make_filter(Interval target, Interval bounds, int degree, Kernel kernel) {
    FilterPolynomial p;
    p.degree = degree;
    p.target = target;
    p.bounds = bounds;
    p.kernel = kernel;
    p.combined.resize(static_cast<size_t>(degree < 0 ? 0 : degree) + 1);
    check(chebfd_make_filter(target.lo, target.hi, bounds.lo, bounds.hi, degree,
                             static_cast<int>(kernel.kind), kernel.mu, p.combined.data(), &p.alpha,
                             &p.beta));
    return p;
}

inline double eval_scalar(const FilterPolynomial& p, double x) {
    double out = 0.0;
    check(chebfd_eval_scalar(p.combined.data(), p.degree, p.alpha, p.beta, p.bounds.lo, p.bounds.hi,
                             x, &out));
    return out;
}

struct MomentTable {
    Index degree = 0, width = 0;
    std::vector<double> m;
    double& operator()(Index n, Index k) { return m[static_cast<size_t>(n * width + k)]; }
    double operator()(Index n, Index k) const { return m[static_cast<size_t>(n * width + k)]; }
};

template <class S>
std::optional<MomentTable> apply_filter(const SparseMatrix<S>& A, BlockVector<S>& X,
                                        const FilterPolynomial& p, bool want_moments = false) {
    std::optional<MomentTable> mt;
    if (want_moments) {
        mt = MomentTable{p.degree, X.width(),
                         std::vector<double>(static_cast<size_t>((p.degree + 1) * X.width()))};
    }
    check(chebfd_apply_filter(A.get(), X.get(), p.combined.data(), p.degree, p.alpha, p.beta,
                              mt ? mt->m.data() : nullptr));
    return mt;
}

// apply_filter on a HOST block (row-major, this rank's rows), end to end
template <class S>
std::optional<MomentTable> apply_filter_host(const SparseMatrix<S>& A, std::vector<S>& x, Index width,
                                             const FilterPolynomial& p, bool want_moments = false) {
    if (width < 1 || static_cast<Index>(x.size()) != A.info().local_rows * width)
        throw std::invalid_argument("apply_filter_host: x must hold local_rows x width entries");
    if (p.degree >= 2 && static_cast<Index>(p.combined.size()) < p.degree + 1)
        throw std::invalid_argument("apply_filter: coefficient array shorter than degree+1");
    std::optional<MomentTable> mt;
    if (want_moments)
        mt = MomentTable{p.degree, width, std::vector<double>(static_cast<size_t>((p.degree + 1) * width))};
    check(chebfd_apply_filter_host(A.get(), x.data(), width, p.combined.data(), p.degree, p.alpha,
                                   p.beta, mt ? mt->m.data() : nullptr));
    return mt;
}

// A stream of host blocks filtered with the copies of neighbouring jobs overlapped
// (chebfd_filter_pipe_*).  Buffers must outlive wait(); results = apply_filter_host's.
template <class S>
class FilterPipe {
  public:
    FilterPipe(const SparseMatrix<S>& A, Index width) { check(chebfd_filter_pipe_create(A.get(), width, &h_)); }
    ~FilterPipe() {
        if (h_) chebfd_filter_pipe_destroy(h_);
    }
    FilterPipe(const FilterPipe&) = delete;
    FilterPipe& operator=(const FilterPipe&) = delete;
    void submit(const S* in, S* out, const FilterPolynomial& p) {
        check(chebfd_filter_pipe_submit(h_, in, out, p.combined.data(), p.degree, p.alpha, p.beta));
    }
    // ... and the Gram X^H X of the filtered block into gram (width x width, row-major)
    void submit(const S* in, S* out, const FilterPolynomial& p, S* gram) {
        check(chebfd_filter_pipe_submit_gram(h_, in, out, p.combined.data(), p.degree, p.alpha,
                                             p.beta, gram));
    }
    void wait() { check(chebfd_filter_pipe_wait(h_)); }

  private:
    chebfd_filter_pipe* h_ = nullptr;
};

// ---- spectral (spectral.hpp) ----------------------------------------------------------------
inline Interval lanczos_bounds_of(chebfd_matrix* a, int iters, std::uint64_t seed) {
    Interval b;
    check(chebfd_lanczos_bounds(a, iters, seed, &b.lo, &b.hi));
    return b;
}

// lanczos_bounds (spectral.cpp:96-154)
template <class S>
Interval lanczos_bounds(const SparseMatrix<S>& A, int iters, std::uint64_t seed = 1) {
    return lanczos_bounds_of(A.get(), iters, seed);
}

// ChebSeriesDensity (spectral.hpp:14-33): raw moments on [a, b], Jackson-damped
// reconstruction (density) and closed-form integral (count)
class ChebSeriesDensity {
  public:
    ChebSeriesDensity() = default;
    ChebSeriesDensity(std::vector<double> moments, Interval bounds)
        : moments_(std::move(moments)), bounds_(bounds) {
        if (moments_.empty()) throw std::invalid_argument("ChebSeriesDensity: no moments");
        if (!(bounds.lo < bounds.hi)) throw std::invalid_argument("ChebSeriesDensity: bad bounds");
    }
    const std::vector<double>& moments() const { return moments_; }
    Interval bounds() const { return bounds_; }
    int order() const { return static_cast<int>(moments_.size()) - 1; }
    double density(double lambda) const {
        double out = 0.0;
        check(chebfd_dos_density(moments_.data(), order(), bounds_.lo, bounds_.hi, lambda, &out));
        return out;
    }
    double count(double lo, double hi) const {
        double out = 0.0;
        check(chebfd_dos_count(moments_.data(), order(), bounds_.lo, bounds_.hi, lo, hi, &out));
        return out;
    }
    double total() const { return moments_.empty() ? 0.0 : moments_[0]; }

  private:
    std::vector<double> moments_;
    Interval bounds_;
};

// DosEstimate (spectral.hpp:36-56)
class DosEstimate {
  public:
    DosEstimate() = default;
    DosEstimate(std::vector<double> moments, Interval bounds, int num_samples, Index dim)
        : series_(std::move(moments), bounds), num_samples_(num_samples), dim_(dim) {}
    double density(double lambda) const { return series_.density(lambda); }
    double count(double lo, double hi) const { return series_.count(lo, hi); }
    Interval bounds() const { return series_.bounds(); }
    const std::vector<double>& moments() const { return series_.moments(); }
    int num_samples() const { return num_samples_; }
    Index matrix_dim() const { return dim_; }

  private:
    ChebSeriesDensity series_;
    int num_samples_ = 0;
    Index dim_ = 0;
};

// WeightDensity (spectral.hpp:57-72): integrates to N_S over the full interval
class WeightDensity {
  public:
    WeightDensity() = default;
    WeightDensity(std::vector<double> moments, Interval bounds) : series_(std::move(moments), bounds) {}
    double density(double lambda) const { return series_.density(lambda); }
    double count(double lo, double hi) const { return series_.count(lo, hi); }
    double integral() const { return series_.total(); }
    Interval bounds() const { return series_.bounds(); }
    const std::vector<double>& moments() const { return series_.moments(); }

  private:
    ChebSeriesDensity series_;
};

// weight_density (spectral.cpp:81-88)
inline WeightDensity weight_density(const MomentTable& moments, Interval bounds) {
    if (moments.width == 0 || moments.m.empty())
        throw std::invalid_argument("weight_density: empty moment table");
    std::vector<double> mu(static_cast<size_t>(moments.degree) + 1);
    check(chebfd_weight_density(moments.m.data(), static_cast<int>(moments.degree), moments.width,
                                mu.data()));
    return WeightDensity(std::move(mu), bounds);
}

// kpm_dos (spectral.cpp:156-205): stochastic-trace KPM DOS on the device
template <class S>
DosEstimate kpm_dos(const SparseMatrix<S>& A, Interval bounds, int order, int num_samples,
                    std::uint64_t seed = 1) {
    std::vector<double> mu(static_cast<size_t>(order < 0 ? 0 : order) + 1);
    check(chebfd_kpm_dos(A.get(), bounds.lo, bounds.hi, order, num_samples, seed, mu.data()));
    return DosEstimate(std::move(mu), bounds, num_samples, A.dim());
}

// estimate_count (spectral.cpp:90-94)
inline double estimate_count(const DosEstimate& dos, Interval interval) {
    if (!dos.bounds().contains(interval))
        throw std::invalid_argument("estimate_count: interval outside DOS bounds");
    return dos.count(interval.lo, interval.hi);
}

// ---- solver (solver.hpp) ------------------------------------------------------------------------
struct SolverOptions {
    Interval target;
    double epsilon = 1e-10;
    int n_search = 0;
    int degree = 0;
    Kernel kernel{KernelKind::Lanczos, 2};
    int max_iters = 40;
    std::uint64_t seed = 1;
    int dos_moments = 2000;
    int dos_samples = 32;
    bool deterministic = true;
    Interval bounds{0.0, 0.0};
    bool collect_weight_density = true;
};

// RitzSet (solver.hpp:27-33)
template <class S>
struct RitzSet {
    std::vector<double> values;          // ascending
    BlockVector<S> vectors;              // orthonormal columns (device)
    std::vector<double> residual_norms;  // ||A v - lambda v||
    std::vector<bool> accepted;
};

struct IterationStat {
    int iteration = 0;
    double min_residual = 0.0;
    double max_residual = 0.0;
    int accepted_count = 0;
    double cumulative_spmvms = 0.0;
};

// ConvergenceReport (solver.hpp:43-60)
template <class S>
struct ConvergenceReport {
    bool converged = false;
    int iterations = 0;
    double total_spmvms = 0.0;
    int n_search = 0;
    int degree = 0;
    double sigma = 0.0;
    double eta = 0.0;
    Interval bounds;
    double matrix_norm_est = 0.0;
    double n_target_estimate = 0.0;
    RitzSet<S> ritz;
    std::vector<IterationStat> history;
    WeightDensity weight;
    bool have_weight = false;
    double seconds = 0.0;
};

// SvqbResult / svqb_orthonormalize (solver.hpp:64-71, solver.cpp:32-61)
template <class S>
struct SvqbResult {
    BlockVector<S> q;
    Index rank = 0;
};

template <class S>
SvqbResult<S> svqb_orthonormalize(const BlockVector<S>& y, double drop_tol = 1e-14) {
    BlockVector<S> q(y, y.width());
    std::int64_t rank = 0;
    check(chebfd_svqb(y.get(), drop_tol, q.get(), &rank));
    SvqbResult<S> out;
    out.rank = rank;
    if (rank == y.width()) {
        out.q = std::move(q);
    } else {  // the reference returns exactly `rank` columns
        BlockVector<S> qr(y, rank);
        check(chebfd_block_copy_columns(qr.get(), 0, q.get(), 0, rank));
        out.q = std::move(qr);
    }
    return out;
}

// rayleigh_ritz (solver.hpp:73-75, solver.cpp:63-91)
template <class S>
RitzSet<S> rayleigh_ritz(const SparseMatrix<S>& A, const BlockVector<S>& q) {
    RitzSet<S> r;
    r.vectors = BlockVector<S>(q, q.width());
    r.values.resize(static_cast<size_t>(q.width()));
    r.residual_norms.resize(static_cast<size_t>(q.width()));
    check(chebfd_rayleigh_ritz(A.get(), q.get(), r.vectors.get(), r.values.data(),
                               r.residual_norms.data()));
    r.accepted.assign(static_cast<size_t>(q.width()), false);
    return r;
}

// solve (solver.hpp:77-80, solver.cpp:93-214): the host loop of the reference with
// every block operation on the device
template <class S>
ConvergenceReport<S> solve(const SparseMatrix<S>& A, const SolverOptions& o) {
    chebfd_solver_options c{};
    chebfd_solver_options_default(&c);
    c.target_lo = o.target.lo;
    c.target_hi = o.target.hi;
    c.epsilon = o.epsilon;
    c.n_search = o.n_search;
    c.degree = o.degree;
    c.kernel = static_cast<int>(o.kernel.kind);
    c.kernel_mu = o.kernel.mu;
    c.max_iters = o.max_iters;
    c.seed = o.seed;
    c.dos_moments = o.dos_moments;
    c.dos_samples = o.dos_samples;
    c.bounds_lo = o.bounds.lo;
    c.bounds_hi = o.bounds.hi;
    c.collect_weight_density = o.collect_weight_density ? 1 : 0;
    chebfd_solve_report r{};
    const int cap = 4096 + 2 * o.n_search;
    std::vector<double> vals(cap), res(cap), hist(static_cast<size_t>(5 * std::max(o.max_iters, 1)));
    std::vector<int> acc(cap);
    const int wcap = 1 << 20;
    std::vector<double> wmu(wcap);
    int wlen = 0;
    chebfd_block* vh = nullptr;
    check(chebfd_solve_ex(A.get(), &c, &r, cap, vals.data(), res.data(), acc.data(), hist.data(),
                          &vh, wcap, wmu.data(), &wlen));
    ConvergenceReport<S> out;
    out.converged = r.converged != 0;
    out.iterations = r.iterations;
    out.total_spmvms = r.total_spmvms;
    out.n_search = r.n_search;
    out.degree = r.degree;
    out.sigma = r.sigma;
    out.eta = r.eta;
    out.bounds = {r.bounds_lo, r.bounds_hi};
    out.matrix_norm_est = r.matrix_norm_est;
    out.n_target_estimate = r.n_target_estimate;
    out.ritz.values.assign(vals.begin(), vals.begin() + r.n_values);
    out.ritz.residual_norms.assign(res.begin(), res.begin() + r.n_values);
    for (int k = 0; k < r.n_values; ++k) out.ritz.accepted.push_back(acc[k] != 0);
    if (vh) out.ritz.vectors = BlockVector<S>(vh);
    for (int i = 0; i < r.iterations; ++i) {
        const double* h = hist.data() + 5 * i;
        out.history.push_back({static_cast<int>(h[0]), h[1], h[2], static_cast<int>(h[3]), h[4]});
    }
    if (wlen > 0) {
        out.weight = WeightDensity(std::vector<double>(wmu.begin(), wmu.begin() + wlen), out.bounds);
        out.have_weight = true;
    }
    out.seconds = r.seconds;
    return out;
}

}  // namespace chebfd::b200
