// Helpers shared by the C-ABI translation units (capi.cu, solver.cu, blas.cu).
#pragma once
#include <atomic>
#include <exception>
#include <functional>
#include <thread>

#include <string>

#include "internal.hpp"

namespace cfd {

extern thread_local std::string g_last_error;

// Run f, translating internal exceptions into status codes (ABI boundary).
template <class F>
int guard(F&& f) {
    try {
        f();
        return CHEBFD_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_last_error = std::string("host allocation failed: ") + e.what();
        return CHEBFD_ERR_RUNTIME;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return CHEBFD_ERR_RUNTIME;
    }
}

void cublas_check(int st, const char* what);
void nccl_check(int st, const char* what);
void ctx_sync(Context& c);
// zero = false: only the halo rows are cleared (for blocks every owned row of
// which the caller overwrites before reading)
std::unique_ptr<Block> make_block(Context& c, const Matrix* m, int kind, int64_t rows,
                                  int64_t width, bool zero = true);
void check_same_shape(const Block& x, const Block& y);
// BlockVector::randomize of this rank's rows, streamed host -> device
void randomize_upload(Context& c, Block& b, uint64_t seed);
// the same on a helper thread (own stream and pinned buffers); b is ready after join()
class AsyncRandomize {
  public:
    AsyncRandomize(Context& c, Block& b, uint64_t seed);
    ~AsyncRandomize();
    AsyncRandomize(const AsyncRandomize&) = delete;
    AsyncRandomize& operator=(const AsyncRandomize&) = delete;
    void join();

  private:
    std::thread th_;
    std::exception_ptr err_;
    std::atomic<bool> cancel_{false};
};
void check_conforms(const Matrix& a, const Block& x, const char* who);
// moments by the Chebyshev doubling identities (CHEBFD_OPT_MOMENTS, Hermitian operators)
bool moment_doubling(const Context& c, const Matrix& a);
void run_step_all(Context& c, const Matrix& a, StepArgs s, Block& gathered);
// interior + boundary launches of a step whose halo exchange is enqueued (c.ev_b)
void launch_split(Context& c, const Matrix& a, StepArgs s);
const void* gather_base(const Matrix& a, const Block& b);
void ensure_halo_buffers(Context& c, Matrix& a, int64_t width);
void build_matrix_device(Context& c, Matrix& m, const HostCsr& csr);
Context* create_group_context(int device, int rank, int nranks);
struct VGroup;
void vgroup_purge(VGroup& g, const void* a, const void* x);
void destroy_group_context(Context* c);
void setup_partition(Context& c, Matrix& m, const HostCsr& csr, int64_t r0, int64_t r1,
                     const std::vector<int64_t>& starts, bool compact);
void ensure_scaled_values(Context& ctx, Matrix& a, double s, cudaStream_t st);
void purge_graphs(Context& c, const void* a, const void* x);
struct FilterWorkspace;
FilterWorkspace& filter_workspace(Context& c, const Matrix& a, int64_t width, bool moments);
bool moment_doubling(const Context& c, const Matrix& a);
// apply_filter's step sequence (filter.hpp:73-116) as calls run(step args, gathered block)
void enqueue_filter(Context& c, const Matrix& a, Block& x, int degree, double alpha, double beta,
                    const double* coeff_dev, double* mom_dev, FilterWorkspace& ws,
                    const std::function<void(const StepArgs&, Block&)>& run);
void allreduce_sum(Context& c, double* dev, size_t n, cudaStream_t st);
void column_dots_host(Context& c, const Block& x, const Block& y, void* out);
void gram_host(Context& c, const Block& x, const Block& y, void* out, bool herm = false);
void apply_filter_device(Context& c, const Matrix& a, Block& x, const double* combined, int degree,
                         double alpha, double beta, double* moments_host);

// blas.cu: cuBLAS / cuSOLVER wrappers on row-major blocks
// dev_out (row-major nx x ny, local rows only) = X^H Y
// herm: the product is known Hermitian (Rayleigh-Ritz Q^H A Q) -- only its upper half
// need be computed
void gemm_gram(Context& c, const Block& x, const Block& y, void* dev_out, bool herm = false);
// the same on the FP64 tensor cores, hand-written (gram.cu)
void gram_dmma(Context& c, const Block& x, const Block& y, void* dev_out, bool herm);
// Y = X B (complex, B row-major nb x bcols on the device) on the FP64 tensor cores (gram.cu)
void tsgemm_dmma(Context& c, const Block& x, const void* b_dev, int64_t bcols, Block& y);
// Y = X B with B given on the host (row-major nb x bcols)
void mult_small_host_b(Context& c, const Block& x, const void* b_host, int64_t bcols, Block& y);
// Y = X B with B on the device (row-major)
void mult_small_dev_b(Context& c, const Block& x, const void* b_dev, int64_t bcols, Block& y);
// Hermitian eigendecomposition of a host row-major n x n matrix (already
// symmetrised): ascending eigenvalues, row-major eigenvectors (columns).
// Returns false if the solver reports failure.
bool heev_host(Context& c, int kind, int64_t n, const void* a_rowmajor, double* w, void* v_rowmajor,
               bool vectors);
void destroy_cusolver(Context& c);

}  // namespace cfd
