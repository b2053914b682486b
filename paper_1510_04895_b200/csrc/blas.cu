// Dense pieces of Rayleigh-Ritz / SVQB on row-major device blocks:
// tall-skinny Gram (X^H Y) and block rotation (X B) through cuBLAS (FP64
// DMMA on sm_100), small Hermitian eigensolves through cuSOLVER.
//
// Row-major D x nb block == column-major nb x D matrix, so
//   G = X^H Y  (row-major nx x ny)  ==  col-major  Y * X^H   (ny x nx)
//   Y = X B    (row-major)          ==  col-major  B_c * X_c (bcols x D)
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <complex>
#include <vector>

#include "capi_common.hpp"

namespace cfd {

namespace {
cublasHandle_t blas(Context& c) { return reinterpret_cast<cublasHandle_t>(c.cublas); }

cusolverDnHandle_t solver(Context& c) {
    if (!c.cusolver) {
        cusolverDnHandle_t h;
        if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS)
            fail(CHEBFD_ERR_CUDA, "cusolverDnCreate failed");
        if (cusolverDnSetStream(h, c.stream) != CUSOLVER_STATUS_SUCCESS)
            fail(CHEBFD_ERR_CUDA, "cusolverDnSetStream failed");
        c.cusolver = reinterpret_cast<cusolverDnContext*>(h);
    }
    return reinterpret_cast<cusolverDnHandle_t>(c.cusolver);
}
}  // namespace

void destroy_cusolver(Context& c) {
    if (c.cusolver) cusolverDnDestroy(reinterpret_cast<cusolverDnHandle_t>(c.cusolver));
    c.cusolver = nullptr;
}

void gemm_gram(Context& c, const Block& x, const Block& y, void* dev_out, bool herm) {
    const int nx = static_cast<int>(x.width), ny = static_cast<int>(y.width);
    const int64_t rows = x.rows;
    if (nx == 0 || ny == 0) return;
    if (rows == 0) {
        CFD_CUDA(cudaMemsetAsync(dev_out, 0, static_cast<size_t>(nx) * ny * x.scalar_bytes(), c.stream));
        return;
    }
    // the hand-written FP64 tensor-core kernel (gram.cu) for complex blocks of 48+ columns
    // (measured: at par with cuBLAS on one 64-column super-tile, its Hermitian half pays at
    // n_b = 256); cuBLAS for real and narrow blocks, where its kernels are faster
    // (tools/gram_exp.py, profiles/r02_gram_ab.jsonl); CHEBFD_OPT_GRAM = 2 forces it
    if ((c.gram_mode == 1 && x.kind == CHEBFD_COMPLEX128 && std::min(nx, ny) >= 48) ||
        (c.gram_mode == 2 && (x.kind == CHEBFD_COMPLEX128 || (nx % 2 == 0 && ny % 2 == 0)))) {
        gram_dmma(c, x, y, dev_out, herm);
        return;
    }
    require(rows < (1LL << 31), "gram: row count exceeds the cuBLAS 32-bit k dimension");
    if (x.kind == CHEBFD_REAL64) {
        const double one = 1.0, zero = 0.0;
        cublas_check(cublasDgemm(blas(c), CUBLAS_OP_N, CUBLAS_OP_T, ny, nx, static_cast<int>(rows),
                                 &one, static_cast<const double*>(y.owned()), ny,
                                 static_cast<const double*>(x.owned()), nx, &zero,
                                 static_cast<double*>(dev_out), ny),
                     "cublasDgemm(gram)");
    } else {
        const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
        cublas_check(cublasZgemm(blas(c), CUBLAS_OP_N, CUBLAS_OP_C, ny, nx, static_cast<int>(rows),
                                 &one, static_cast<const cuDoubleComplex*>(y.owned()), ny,
                                 static_cast<const cuDoubleComplex*>(x.owned()), nx, &zero,
                                 static_cast<cuDoubleComplex*>(dev_out), ny),
                     "cublasZgemm(gram)");
    }
    c.launches++;
}

void mult_small_dev_b(Context& c, const Block& x, const void* b_dev, int64_t bcols, Block& y) {
    const int nb = static_cast<int>(x.width), m = static_cast<int>(bcols);
    const int64_t rows = x.rows;
    if (rows == 0 || m == 0) return;
    if (nb == 0) {
        CFD_CUDA(cudaMemsetAsync(y.owned(), 0, y.owned_bytes(), c.stream));
        return;
    }
    // complex rotations of 48+ columns on the hand-written DMMA kernel (gram.cu), as the Gram
    if (x.kind == CHEBFD_COMPLEX128 && c.gram_mode >= 1 && (std::min(nb, m) >= 48 || c.gram_mode == 2)) {
        tsgemm_dmma(c, x, b_dev, bcols, y);
        return;
    }
    require(rows < (1LL << 31), "block_mult_small: row count exceeds 32-bit n dimension");
    if (x.kind == CHEBFD_REAL64) {
        const double one = 1.0, zero = 0.0;
        cublas_check(cublasDgemm(blas(c), CUBLAS_OP_N, CUBLAS_OP_N, m, static_cast<int>(rows), nb,
                                 &one, static_cast<const double*>(b_dev), m,
                                 static_cast<const double*>(x.owned()), nb, &zero,
                                 static_cast<double*>(y.owned()), m),
                     "cublasDgemm(mult_small)");
    } else {
        const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
        cublas_check(cublasZgemm(blas(c), CUBLAS_OP_N, CUBLAS_OP_N, m, static_cast<int>(rows), nb,
                                 &one, static_cast<const cuDoubleComplex*>(b_dev), m,
                                 static_cast<const cuDoubleComplex*>(x.owned()), nb, &zero,
                                 static_cast<cuDoubleComplex*>(y.owned()), m),
                     "cublasZgemm(mult_small)");
    }
    c.launches++;
}

void mult_small_host_b(Context& c, const Block& x, const void* b_host, int64_t bcols, Block& y) {
    const size_t bytes = static_cast<size_t>(x.width * bcols) * x.scalar_bytes();
    DeviceBuffer& b = c.small[2];
    b.ensure(std::max<size_t>(bytes, 16));
    if (bytes)
        CFD_CUDA(cudaMemcpyAsync(b.p, b_host, bytes, cudaMemcpyHostToDevice, c.stream));
    mult_small_dev_b(c, x, b.p, bcols, y);
    ctx_sync(c);  // b_host may be released by the caller
}

bool heev_host(Context& c, int kind, int64_t n64, const void* a_rowmajor, double* w, void* v_rowmajor,
               bool vectors) {
    const int n = static_cast<int>(n64);
    if (n == 0) return true;
    cusolverDnHandle_t h = solver(c);
    const size_t sb = kind ? 16 : 8;
    // column-major copy of A
    std::vector<double> acol(static_cast<size_t>(n) * n * (kind ? 2 : 1));
    const double* a = static_cast<const double*>(a_rowmajor);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            if (kind) {
                acol[2 * (i + static_cast<size_t>(j) * n)] = a[2 * (static_cast<size_t>(i) * n + j)];
                acol[2 * (i + static_cast<size_t>(j) * n) + 1] = a[2 * (static_cast<size_t>(i) * n + j) + 1];
            } else {
                acol[i + static_cast<size_t>(j) * n] = a[static_cast<size_t>(i) * n + j];
            }
        }
    DeviceBuffer& da = c.small[3];
    da.ensure(sb * n * n + sizeof(double) * n + 16);
    double* dw_p = reinterpret_cast<double*>(static_cast<char*>(da.p) + sb * n * n);
    int* dinfo_p = reinterpret_cast<int*>(dw_p + n);
    CFD_CUDA(cudaMemcpyAsync(da.p, acol.data(), sb * n * n, cudaMemcpyHostToDevice, c.stream));
    const cusolverEigMode_t mode = vectors ? CUSOLVER_EIG_MODE_VECTOR : CUSOLVER_EIG_MODE_NOVECTOR;
    int lwork = 0;
    if (kind == CHEBFD_REAL64) {
        if (cusolverDnDsyevd_bufferSize(h, mode, CUBLAS_FILL_MODE_LOWER, n, da.as<double>(), n,
                                        dw_p, &lwork) != CUSOLVER_STATUS_SUCCESS)
            fail(CHEBFD_ERR_CUDA, "cusolverDnDsyevd_bufferSize failed");
        c.workspace.ensure(sizeof(double) * std::max(lwork, 1));
        if (cusolverDnDsyevd(h, mode, CUBLAS_FILL_MODE_LOWER, n, da.as<double>(), n, dw_p,
                             c.workspace.as<double>(), lwork, dinfo_p) != CUSOLVER_STATUS_SUCCESS)
            fail(CHEBFD_ERR_CUDA, "cusolverDnDsyevd failed");
    } else {
        if (cusolverDnZheevd_bufferSize(h, mode, CUBLAS_FILL_MODE_LOWER, n, da.as<cuDoubleComplex>(), n,
                                        dw_p, &lwork) != CUSOLVER_STATUS_SUCCESS)
            fail(CHEBFD_ERR_CUDA, "cusolverDnZheevd_bufferSize failed");
        c.workspace.ensure(sizeof(cuDoubleComplex) * std::max(lwork, 1));
        if (cusolverDnZheevd(h, mode, CUBLAS_FILL_MODE_LOWER, n, da.as<cuDoubleComplex>(), n,
                             dw_p, c.workspace.as<cuDoubleComplex>(), lwork,
                             dinfo_p) != CUSOLVER_STATUS_SUCCESS)
            fail(CHEBFD_ERR_CUDA, "cusolverDnZheevd failed");
    }
    c.launches++;
    int info = 0;
    CFD_CUDA(cudaMemcpyAsync(&info, dinfo_p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    CFD_CUDA(cudaMemcpyAsync(w, dw_p, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
    if (vectors)
        CFD_CUDA(cudaMemcpyAsync(acol.data(), da.p, sb * n * n, cudaMemcpyDeviceToHost, c.stream));
    ctx_sync(c);
    if (info != 0) return false;
    if (vectors) {
        double* v = static_cast<double*>(v_rowmajor);
        for (int i = 0; i < n; ++i)
            for (int k = 0; k < n; ++k) {
                if (kind) {
                    v[2 * (static_cast<size_t>(i) * n + k)] = acol[2 * (i + static_cast<size_t>(k) * n)];
                    v[2 * (static_cast<size_t>(i) * n + k) + 1] = acol[2 * (i + static_cast<size_t>(k) * n) + 1];
                } else {
                    v[static_cast<size_t>(i) * n + k] = acol[i + static_cast<size_t>(k) * n];
                }
            }
    }
    return true;
}

}  // namespace cfd
