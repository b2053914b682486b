// Tall-skinny Gram G = X^H Y and block rotation Y = X B on FP64 tensor cores (DMMA),
// hand-written for sm_100a.
//
// gram (kernels.hpp:165-192) is G(k,l) = <x_k, y_l> over D rows of two row-major blocks
// of widths nx, ny <= a few hundred: a GEMM with a huge K (D up to 67 M) and a small
// output.  Here:
//  * the output is cut into 64 x 64 super-tiles; for Y^H Y (X and Y the same block:
//    SVQB's Gram, solver.cpp:35) only super-tiles on or above the diagonal are computed
//    and the lower ones mirrored (conjugate transpose) -- 10 of 16 at n_b = 256;
//  * split-K: CTA (tile, s) sums rows [s D / S, (s+1) D / S); partial tiles are summed in
//    split order by a second kernel (fixed order: bitwise reproducible);
//  * 8 warps per CTA, 2 CTAs per SM: 16-row stages of both operands' 64-column slabs
//    arrive by cp.async (16-byte copies, three stages in flight) in the blocks' own
//    interleaved layout; complex fragments are single 16-byte shared loads (re and im
//    together); a diagonal super-tile of Y^H Y stages its slab once;
//  * every warp owns a 16 x 32 region of the super-tile: 2 x 4 m8n8k4 tiles, complex
//    products as four real DMMAs, Re += Xr^T Yr + Xi^T Yi, Im += Xr^T Yi - Xi^T Yr
//    (mma.sync.aligned.m8n8k4.row.col.f64: FP64 tensor pipe, DMMA in SASS).
// Summation order differs from the reference's Kahan chunks; the tests hold it to
// 1e-13 of the largest entry.
#include <cuda_runtime.h>

#include <algorithm>

#include "capi_common.hpp"

namespace cfd {

namespace {

constexpr int kTS = 64;        // super-tile edge
constexpr int kKS = 16;        // rows per pipeline stage
constexpr int kNST = 3;        // stages in flight (cp.async)
constexpr int kThreads = 256;
// shared row pitch in scalars: complex rows are read with 16-byte fragments (8 columns
// x 16 B = one 128-byte wavefront per k-row, conflict-free); real rows with 8-byte ones,
// padded by 8 doubles so the 4 k-rows of a fragment fill two disjoint bank halves
template <bool CPLX>
constexpr int pitch_of() { return CPLX ? kTS : kTS + 8; }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool in) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src),
                 "r"(in ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

struct GramParams {
    const void* x;       // owned rows, row-major, nx (ny) scalars per row
    const void* y;
    int64_t rows;
    int nx, ny;
    const int2* tiles;   // (I0, J0) of each super-tile
    int splits;
    double2* partials;   // [split][tile][kTS][kTS] (real: .y unused)
    int same;            // X and Y are the same block (Y^H Y)
};

template <bool CPLX>
__global__ void __launch_bounds__(kThreads, 2) gram_dmma_kernel(const GramParams p) {
    using S = std::conditional_t<CPLX, double2, double>;
    constexpr int PITCH = pitch_of<CPLX>();
    constexpr int OPSZ = kKS * PITCH;  // scalars per operand per stage
    extern __shared__ __align__(16) unsigned char gsm_raw[];
    S* gsm = reinterpret_cast<S*>(gsm_raw);
    const int tile = blockIdx.x, split = blockIdx.y;
    const int2 tt = p.tiles[tile];
    const int I0 = tt.x, J0 = tt.y;
    const bool diag = p.same && I0 == J0;  // one slab serves both operands
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t r_beg = p.rows * split / p.splits, r_end = p.rows * (split + 1) / p.splits;
    const S* X = static_cast<const S*>(p.x);
    const S* Y = static_cast<const S*>(p.y);
    auto xs = [&](int st) { return gsm + (2 * st) * OPSZ; };
    auto ys = [&](int st) { return gsm + (2 * st + 1) * OPSZ; };
    // stage `st` <- rows [r0, r0 + kKS) of the two 64-column slabs; 16-byte copies, zero
    // filled outside the rows / columns (cp.async src-size 0)
    constexpr int PER16 = 16 / sizeof(S);              // scalars per 16-byte copy
    constexpr int COPIES = kKS * kTS / PER16;          // per operand per stage
    auto issue = [&](int st, int64_t r0) {
        for (int q = t; q < COPIES; q += kThreads) {
            const int row = q / (kTS / PER16), c = (q - row * (kTS / PER16)) * PER16;
            const int64_t r = r0 + row;
            const bool rin = r < r_end;
            const int cx = I0 + c, cy = J0 + c;
            // a 16-byte copy of a real operand covers two columns: nx, ny even (below)
            cp_async16(xs(st) + row * PITCH + c, X + (rin && cx < p.nx ? r * p.nx + cx : 0),
                       rin && cx < p.nx);
            if (!diag)
                cp_async16(ys(st) + row * PITCH + c, Y + (rin && cy < p.ny ? r * p.ny + cy : 0),
                           rin && cy < p.ny);
        }
    };
    const int m0 = 16 * (w >> 1), n0 = 32 * (w & 1);
    double cre[2][4][2], cim[2][4][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            cre[a][b][0] = cre[a][b][1] = 0.0;
            cim[a][b][0] = cim[a][b][1] = 0.0;
        }
    const int fk = lane & 3, fm = lane >> 2;
    const int64_t nst = (r_end - r_beg + kKS - 1) / kKS;
#pragma unroll
    for (int s = 0; s < kNST - 1; ++s) {
        if (s < nst) issue(s, r_beg + s * kKS);
        cp_async_commit();
    }
    for (int64_t it = 0; it < nst; ++it) {
        cp_async_wait<kNST - 2>();
        __syncthreads();  // stage it landed for everyone; stage it - 1 is free again
        {
            const int64_t nx_it = it + kNST - 1;
            if (nx_it < nst) issue(static_cast<int>(nx_it % kNST), r_beg + nx_it * kKS);
            cp_async_commit();
        }
        const int st = static_cast<int>(it % kNST);
        const S* xa = xs(st);
        const S* yb = diag ? xa : ys(st);
#pragma unroll
        for (int ks = 0; ks < kKS; ks += 4) {
            const int row = (ks + fk) * PITCH;
            double ar[2], ai[2], br[4], bi[4];
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const S v = xa[row + m0 + 8 * a + fm];
                if constexpr (CPLX) {
                    ar[a] = v.x;
                    ai[a] = v.y;
                } else {
                    ar[a] = v;
                }
            }
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const S v = yb[row + n0 + 8 * b + fm];
                if constexpr (CPLX) {
                    br[b] = v.x;
                    bi[b] = v.y;
                } else {
                    br[b] = v;
                }
            }
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) dmma(cre[a][b], ar[a], br[b]);
            if constexpr (CPLX) {
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) dmma(cim[a][b], ar[a], bi[b]);
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) dmma(cre[a][b], ai[a], bi[b]);
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) dmma(cim[a][b], -ai[a], br[b]);
            }
        }
    }
    cp_async_wait<0>();
    // partial tile: C[m][n], m = m0 + 8a + fm, n = n0 + 8b + 2 fk + {0, 1}
    double2* out = p.partials + (static_cast<size_t>(split) * gridDim.x + tile) * (kTS * kTS);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int m = m0 + 8 * a + fm, n = n0 + 8 * b + 2 * fk + e;
                out[m * kTS + n] = make_double2(cre[a][b][e], cim[a][b][e]);
            }
}

// G = sum over splits (in order) of the partial tiles; lower super-tiles of Y^H Y are
// the conjugate transposes of the upper ones
template <bool CPLX>
__global__ void gram_reduce_kernel(const double2* __restrict__ partials, const int2* __restrict__ tiles,
                                   int ntiles, int splits, int nx, int ny, int same, void* g) {
    const int tile = blockIdx.y;
    const int2 tt = tiles[tile];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < kTS * kTS; e += gridDim.x * blockDim.x) {
        const int m = e / kTS, n = e - m * kTS;
        const int gi = tt.x + m, gj = tt.y + n;
        if (gi >= nx || gj >= ny) continue;
        double re = 0.0, im = 0.0;
        for (int s = 0; s < splits; ++s) {
            const double2 v = partials[(static_cast<size_t>(s) * ntiles + tile) * (kTS * kTS) + e];
            re += v.x;
            im += v.y;
        }
        if constexpr (CPLX) {
            double2* G = static_cast<double2*>(g);
            G[static_cast<int64_t>(gi) * ny + gj] = make_double2(re, im);
            if (same && tt.x != tt.y) G[static_cast<int64_t>(gj) * ny + gi] = make_double2(re, -im);
        } else {
            double* G = static_cast<double*>(g);
            G[static_cast<int64_t>(gi) * ny + gj] = re;
            if (same && tt.x != tt.y) G[static_cast<int64_t>(gj) * ny + gi] = re;
        }
    }
}

// ---- block_mult_small Y = X B (kernels.hpp:216-232) on the FP64 tensor cores ------------
// M = this rank's rows, N = m (B's columns), K = n_b.  CTA tile 64 rows x 64 columns of
// Y, K streamed in 16-wide chunks of X (row-major, pitch 17 complex: the 8 rows x 4 k of
// a fragment fill distinct bank groups) and of B (row-major, L2-resident across tiles);
// the same warp layout and fragments as the Gram: Re += Xr Br - Xi Bi, Im += Xr Bi + Xi Br.
struct TsParams {
    const double2* x;   // rows x nb
    const double2* b;   // nb x m, row-major
    double2* y;         // rows x m
    int64_t rows;
    int nb, m;
};

constexpr int kXP = kKS + 1;  // X tile row pitch (complex): fragment rows fall in distinct banks
constexpr int kTsStage = kTS * kXP + kKS * kTS;  // complex entries per stage (X tile + B chunk)

__global__ void __launch_bounds__(kThreads, 2) tsgemm_dmma_kernel(const TsParams p) {
    extern __shared__ __align__(16) unsigned char tsm_raw[];
    double2* sm = reinterpret_cast<double2*>(tsm_raw);
    // stage st: X tile [64 rows][kXP] row-major (as in global), B chunk [kKS][64]
    auto xs = [&](int st) { return sm + st * kTsStage; };
    auto bs = [&](int st) { return sm + st * kTsStage + kTS * kXP; };
    const int64_t R0 = static_cast<int64_t>(blockIdx.x) * kTS;
    const int N0 = blockIdx.y * kTS;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    auto issue = [&](int st, int K0) {
        for (int q = t; q < kKS * kTS; q += kThreads) {
            // X: row i, k-column kk of the chunk -> xs[i][kk] (coalesced along k)
            const int i = q / kKS, kk = q - i * kKS;
            const int64_t r = R0 + i;
            const bool xin = r < p.rows && K0 + kk < p.nb;
            cp_async16(xs(st) + i * kXP + kk, p.x + (xin ? r * p.nb + K0 + kk : 0), xin);
            // B: k-row bk, column n -> bs[bk][n]
            const int bk = q / kTS, n = q - bk * kTS;
            const bool bin = K0 + bk < p.nb && N0 + n < p.m;
            cp_async16(bs(st) + bk * kTS + n, p.b + (bin ? static_cast<int64_t>(K0 + bk) * p.m + N0 + n : 0),
                       bin);
        }
    };
    const int m0 = 16 * (w >> 1), n0 = 32 * (w & 1);
    double cre[2][4][2], cim[2][4][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            cre[a][b][0] = cre[a][b][1] = 0.0;
            cim[a][b][0] = cim[a][b][1] = 0.0;
        }
    const int fk = lane & 3, fm = lane >> 2;
    const int nst = (p.nb + kKS - 1) / kKS;
#pragma unroll
    for (int s = 0; s < kNST - 1; ++s) {
        if (s < nst) issue(s, s * kKS);
        cp_async_commit();
    }
    for (int it = 0; it < nst; ++it) {
        cp_async_wait<kNST - 2>();
        __syncthreads();
        if (it + kNST - 1 < nst) issue((it + kNST - 1) % kNST, (it + kNST - 1) * kKS);
        cp_async_commit();
        const double2* xa = xs(it % kNST);
        const double2* bb = bs(it % kNST);
#pragma unroll
        for (int ks = 0; ks < kKS; ks += 4) {
            const int row = (ks + fk) * kTS;
            double ar[2], ai[2], br[4], bi[4];
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const double2 v = xa[(m0 + 8 * a + fm) * kXP + ks + fk];
                ar[a] = v.x;
                ai[a] = v.y;
            }
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const double2 v = bb[row + n0 + 8 * b + fm];
                br[b] = v.x;
                bi[b] = v.y;
            }
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) dmma(cre[a][b], ar[a], br[b]);
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) dmma(cim[a][b], ar[a], bi[b]);
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) dmma(cre[a][b], -ai[a], bi[b]);
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) dmma(cim[a][b], ai[a], br[b]);
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int64_t r = R0 + m0 + 8 * a + fm;
                const int n = N0 + n0 + 8 * b + 2 * fk + e;
                if (r < p.rows && n < p.m) p.y[r * p.m + n] = make_double2(cre[a][b][e], cim[a][b][e]);
            }
}

}  // namespace

// Y = X B (complex blocks, B on the device, row-major nb x m) on the FP64 tensor cores.
void tsgemm_dmma(Context& c, const Block& x, const void* b_dev, int64_t bcols, Block& y) {
    const int nb = static_cast<int>(x.width), m = static_cast<int>(bcols);
    require(x.kind == CHEBFD_COMPLEX128, "tsgemm_dmma: complex blocks only");
    if (x.rows == 0 || m == 0) return;
    TsParams p{static_cast<const double2*>(x.owned()), static_cast<const double2*>(b_dev),
               static_cast<double2*>(y.owned()), x.rows, nb, m};
    const size_t smem = static_cast<size_t>(kNST) * kTsStage * sizeof(double2);
    static bool attr = false;
    if (!attr) {
        CFD_CUDA(cudaFuncSetAttribute(tsgemm_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        attr = true;
    }
    const dim3 grid(static_cast<unsigned>((x.rows + kTS - 1) / kTS), static_cast<unsigned>((m + kTS - 1) / kTS));
    tsgemm_dmma_kernel<<<grid, kThreads, smem, c.stream>>>(p);
    CFD_CUDA(cudaGetLastError());
    c.launches++;
}

// dev_out (row-major nx x ny, this rank's rows) = X^H Y on the FP64 tensor cores.
void gram_dmma(Context& c, const Block& x, const Block& y, void* dev_out, bool herm) {
    const int nx = static_cast<int>(x.width), ny = static_cast<int>(y.width);
    const bool cplx = x.kind == CHEBFD_COMPLEX128;
    if (nx == 0 || ny == 0) return;
    // the product is Hermitian (Y^H Y, or Q^H (A Q) for Hermitian A -- the caller says so):
    // super-tiles on and above the diagonal only, the lower ones mirrored
    const bool same = (herm || x.owned() == y.owned()) && nx == ny;
    const bool one_slab = x.owned() == y.owned();
    // 16-byte staging of real rows covers column pairs: odd real widths (and row bases
    // off 16-byte alignment) take cuBLAS
    require(cplx || (nx % 2 == 0 && ny % 2 == 0), "gram_dmma: odd real width");
    std::vector<int2> tl;
    for (int I = 0; I < nx; I += kTS)
        for (int J = same ? I : 0; J < ny; J += kTS) tl.push_back(make_int2(I, J));
    const int T = static_cast<int>(tl.size());
    const int64_t rows = x.rows;
    int S = std::max(1, (2 * c.num_sms + T - 1) / T);
    S = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(S, (rows + kKS - 1) / kKS)));
    // the super-tile list, uploaded once per shape; the partials scratch grows only
    auto& tb = c.gram_tiles[std::make_tuple(nx, ny, same)];
    if (!tb) {
        tb = std::make_unique<DeviceBuffer>(sizeof(int2) * T);
        CFD_CUDA(cudaMemcpy(tb->p, tl.data(), sizeof(int2) * T, cudaMemcpyHostToDevice));
    }
    int2* d_tiles = tb->as<int2>();
    const size_t pbytes = sizeof(double2) * static_cast<size_t>(S) * T * kTS * kTS;
    c.gram_scratch.ensure(pbytes);
    double2* d_part = c.gram_scratch.as<double2>();
    GramParams p{x.owned(), y.owned(), rows, nx, ny, d_tiles, S, d_part, one_slab ? 1 : 0};
    const size_t smem = static_cast<size_t>(kNST) * 2 /*operands*/ * kKS *
                        (cplx ? pitch_of<true>() * sizeof(double2) : pitch_of<false>() * sizeof(double));
    if (cplx) {
        static bool attr = false;
        if (!attr) {
            CFD_CUDA(cudaFuncSetAttribute(gram_dmma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem)));
            attr = true;
        }
        gram_dmma_kernel<true><<<dim3(T, S), kThreads, smem, c.stream>>>(p);
    } else {
        static bool attr = false;
        if (!attr) {
            CFD_CUDA(cudaFuncSetAttribute(gram_dmma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem)));
            attr = true;
        }
        gram_dmma_kernel<false><<<dim3(T, S), kThreads, smem, c.stream>>>(p);
    }
    CFD_CUDA(cudaGetLastError());
    if (cplx)
        gram_reduce_kernel<true><<<dim3(16, T), 256, 0, c.stream>>>(d_part, d_tiles, T, S, nx, ny,
                                                                    same ? 1 : 0, dev_out);
    // (p.same marks one staged slab for diagonal tiles of Y^H Y; the mirror flag is `same`)
    else
        gram_reduce_kernel<false><<<dim3(16, T), 256, 0, c.stream>>>(d_part, d_tiles, T, S, nx, ny,
                                                                     same ? 1 : 0, dev_out);
    CFD_CUDA(cudaGetLastError());
    c.launches += 2;
}

}  // namespace cfd
