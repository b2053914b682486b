// Device kernels of the ChebFD hot path (sm_100a).
//
// Design:
//  * SELL-C-sigma matrix, C = 32, sigma = 1 (row order kept): entry j of row
//    r lives at chunk_ptr[r/32] + j*32 + r%32, int32 extended-row column
//    index (-1 = padding), value double / double2.
//  * Row-major block vectors.  One THREAD owns one 16-byte unit of a row
//    (one complex entry, or two real columns; 8 bytes for odd real widths);
//    a CTA covers R consecutive rows x U units, so the own-row streams
//    (W, X, x0) are perfectly coalesced and every gathered neighbour row is a
//    contiguous, fully used segment.
//  * Persistent grid (num_SMs x occupancy), rows strided by the grid.
//  * Column dot products: per-thread accumulators -> fixed-order CTA reduction
//    -> per-CTA partials -> the last CTA (ticket counter) reduces the partials
//    in CTA order.  Bitwise run-to-run reproducible.
//  * Arithmetic uses __dmul_rn/__dadd_rn/__dsub_rn in exactly the order of the
//    reference's scalar code (kernels.hpp:46-118 compiled for x86-64 SSE2, no
//    FMA), so W and X match the reference bit for bit; only the dot-product
//    summation order differs (tolerance-checked).
#include <cuda_runtime.h>
#include <curand_kernel.h>

#include <cub/device/device_scan.cuh>
#include <type_traits>

#ifndef CFD_TMA_THREADS
#define CFD_TMA_THREADS 256  // max threads per CTA of the TMA step kernel
#endif
#ifndef CFD_TMA_MINB
#define CFD_TMA_MINB 2  // => 128 registers/thread; CTAs of 64/128 threads then fit 8/4 per SM
#endif
#ifndef CFD_L2_HINTS
// TMA step kernel: gathered rows evict_last, own-row streams evict_first in L2.
// Measured on B200 (tools/l2_exp.py, A/B builds): C2 step 0.581 -> 0.578 ms, C3
// lattice n_b = 32 2.54 -> 2.46 ms, n_b = 256 21.6 -> 21.4 ms, KPM +2 %.
#define CFD_L2_HINTS 1
#endif

#include "internal.hpp"
#include "step_common.cuh"

#include "step_kernels.cuh"

namespace cfd {

namespace {
// values pre-multiplied by s (one rounding per entry, as kernels.hpp:95)
__global__ void scale_values_kernel(double* __restrict__ out, const double* __restrict__ in,
                                    int64_t n, double s) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = mul(in[i], s);
}

// dst row i = src row idx[i] (rows of `words` doubles): the compact halo's send-side pack
// and the virtual group's pull of a neighbour's rows
__global__ void gather_rows_kernel(double* __restrict__ dst, const double* __restrict__ src,
                                   const int64_t* __restrict__ idx, int64_t n, int64_t words) {
    const int64_t tot = n * words;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < tot;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / words, k = i - r * words;
        dst[i] = __ldg(&src[__ldg(&idx[r]) * words + k]);
    }
}
__global__ void gather_rows2_kernel(double2* __restrict__ dst, const double2* __restrict__ src,
                                    const int64_t* __restrict__ idx, int64_t n, int64_t units) {
    const int64_t tot = n * units;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < tot;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / units, k = i - r * units;
        dst[i] = __ldg(&src[__ldg(&idx[r]) * units + k]);
    }
}

// ---- generic per-column reductions ------------------------------------------------------
// mode 0: out_S[k] = sum conj(x) y;  mode 1: out_d[k] = sum |av - lam v|^2
template <bool CPLX, class T, int MODE>
__global__ void __launch_bounds__(256) colreduce_kernel(const T* __restrict__ x,
                                                        const T* __restrict__ y,
                                                        const double* __restrict__ lam,
                                                        int64_t rows, int pitch, int u_off,
                                                        int US, int R, void* out, T* partials,
                                                        unsigned* counter) {
    using O = Ops<CPLX, T>;
    const int t = threadIdx.x;
    const int rr = t / US, u = t - rr * US;
    const int64_t col = u_off + u;
    T acc[1] = {O::zero()};
    for (int64_t rg = blockIdx.x; rg * R < rows; rg += gridDim.x) {
        const int64_t r = rg * R + rr;
        if (r >= rows) continue;
        const T a = ld_stream(&x[r * pitch + col]);
        const T b = ld_stream(&y[r * pitch + col]);
        if constexpr (MODE == 0) {
            acc[0] = O::vadd(acc[0], O::cdot(a, b));
        } else {
            const T res = O::vsub(a, O::lam_mul(lam, static_cast<int>(col) * O::kCols, b));
            acc[0] = O::vadd(acc[0], O::cdot(res, res));
        }
    }
    grid_reduce<T, 1>(acc, R, US, partials, blockIdx.x, gridDim.x, true, counter,
                      [&](int, int uu, T v) {
                          if (MODE == 0)
                              O::store_full(static_cast<T*>(out), u_off + uu, v);
                          else
                              O::store_re(static_cast<double*>(out), u_off + uu, v);
                      });
}

// X = c0 X + c1 U + c2 W on flat doubles (block_axpy_scal, kernels.hpp:147-162)
__global__ void axpy_kernel(double* __restrict__ x, const double* __restrict__ u,
                            const double* __restrict__ w, int64_t n, double c0, double c1,
                            double c2) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] = add(add(mul(c0, x[i]), mul(c1, u[i])), mul(c2, w[i]));
}

// w <- w - h q for single-column blocks (Lanczos reorthogonalisation,
// spectral.cpp:119): real h*q, or GCC's complex expansion of h*q.
__global__ void axpy_scalar_kernel(double* __restrict__ w, const double* __restrict__ q, int64_t n,
                                   int cplx, double hr, double hi) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (!cplx) {
            w[i] = sub(w[i], mul(hr, q[i]));
        } else {
            const double qr = q[2 * i], qi = q[2 * i + 1];
            const double pr = sub(mul(hr, qr), mul(hi, qi));
            const double pi = add(mul(hr, qi), mul(hi, qr));
            w[2 * i] = sub(w[2 * i], pr);
            w[2 * i + 1] = sub(w[2 * i + 1], pi);
        }
    }
}

// x(i,k) /= d[k] on doubles: complex entries divide both parts by d[k]
__global__ void divcols_kernel(double* __restrict__ x, int64_t rows, int64_t width, int cplx,
                               const double* __restrict__ d) {
    const int64_t per_row = width * (cplx ? 2 : 1);
    const int64_t n = rows * per_row;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k = (i % per_row) >> cplx;
        x[i] = div_(x[i], d[k]);
    }
}

__global__ void copycols_kernel(double* __restrict__ dst, int64_t dpitch, int64_t d0,
                                const double* __restrict__ src, int64_t spitch, int64_t s0,
                                int64_t rows, int64_t n) {
    const int64_t tot = rows * n;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < tot;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / n, k = i - r * n;
        dst[r * dpitch + d0 + k] = src[r * spitch + s0 + k];
    }
}

__global__ void philox_normal_kernel(double* __restrict__ x, int64_t n, uint64_t seed) {
    const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    curandStatePhilox4_32_10_t st;
    curand_init(seed, tid, 0, &st);
    for (int64_t i = 2 * tid; i < n; i += 2 * static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double2 g = curand_normal2_double(&st);
        x[i] = g.x;
        if (i + 1 < n) x[i + 1] = g.y;
    }
}

// ---- SELL build --------------------------------------------------------------------------
__global__ void sell_width_kernel(const int64_t* __restrict__ offs, int64_t rows, int64_t nchunks,
                                  int64_t* __restrict__ slots, int* __restrict__ maxlen,
                                  unsigned char* __restrict__ full) {
    const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (c >= nchunks) return;
    int64_t w = 0, wmin = INT64_MAX;
    for (int l = 0; l < kChunk; ++l) {
        const int64_t r = c * kChunk + l;
        const int64_t len = r < rows ? offs[r + 1] - offs[r] : -1;
        w = max(w, len);
        wmin = min(wmin, len);
    }
    slots[c] = w * kChunk;
    full[c] = (wmin == w) ? 1 : 0;  // no padding slot anywhere in the chunk
    atomicMax(maxlen, static_cast<int>(w));
}

#if CFD_EXPERIMENTAL
// Staged-gather plan of one chunk per CTA: sort the extended rows the chunk
// reads (its slots' columns and its own rows), merge them into runs (gaps of
// < kStageGap rows are copied too), and map every slot / own row to its row in
// the concatenated runs.  Overflowing chunks (> kStageRuns runs) flag the
// matrix as unplannable.
__global__ void __launch_bounds__(256) stage_plan_kernel(
    const int64_t* __restrict__ chunk_ptr, const int* __restrict__ cols, int64_t rows,
    int64_t halo_lo, int4* __restrict__ runs_out, int2* __restrict__ meta,
    unsigned short* __restrict__ lcol, unsigned short* __restrict__ lown, int* __restrict__ max_rows,
    int* __restrict__ overflow) {
    __shared__ int v[1024];
    __shared__ int4 runs[kStageRuns];
    __shared__ int nruns_s, nrows_s, bad_s;
    const int64_t c = blockIdx.x;
    const int t = threadIdx.x;
    const int64_t base = chunk_ptr[c];
    const int w = static_cast<int>((chunk_ptr[c + 1] - base) >> 5);
    for (int i = t; i < 1024; i += 256) v[i] = INT_MAX;
    __syncthreads();
    for (int s = t; s < 32 * w && s < 512; s += 256) {
        const int col = cols[base + s];
        v[s] = col >= 0 ? col : INT_MAX;
    }
    if (t < 32) {
        const int64_t r = c * 32 + t;
        v[512 + t] = r < rows ? static_cast<int>(r + halo_lo) : INT_MAX;
    }
    __syncthreads();
    // bitonic sort, 1024 keys
    for (int k = 2; k <= 1024; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = t; i < 1024; i += 256) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k) == 0;
                    const int a = v[i], b = v[ixj];
                    if ((a > b) == up) {
                        v[i] = b;
                        v[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    if (t == 0) {
        int n = 0, rowsum = 0, bad = 0;
        int cs = -1, ce = -1;  // current run [cs, ce]
        for (int i = 0; i < 1024 && v[i] != INT_MAX; ++i) {
            const int e = v[i];
            if (cs >= 0 && e <= ce) continue;  // duplicate
            if (cs >= 0 && e - ce - 1 < kStageGap) {
                ce = e;
                continue;
            }
            if (cs >= 0) {
                if (n < kStageRuns) runs[n] = make_int4(cs, ce - cs + 1, rowsum, 0);
                rowsum += ce - cs + 1;
                ++n;
            }
            cs = ce = e;
        }
        if (cs >= 0) {
            if (n < kStageRuns) runs[n] = make_int4(cs, ce - cs + 1, rowsum, 0);
            rowsum += ce - cs + 1;
            ++n;
        }
        if (n > kStageRuns || rowsum > 65535) bad = 1;
        nruns_s = n;
        nrows_s = rowsum;
        bad_s = bad;
        if (bad) atomicExch(overflow, 1);
        atomicMax(max_rows, rowsum);
        meta[c] = make_int2(bad ? 0 : n, rowsum);
    }
    __syncthreads();
    if (bad_s) return;
    const int n = nruns_s;
    for (int k = t; k < n; k += 256) runs_out[c * kStageRuns + k] = runs[k];
    auto local = [&](int e) -> unsigned short {
        int lo = 0, hi = n - 1;  // last run with start <= e
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (runs[mid].x <= e) lo = mid; else hi = mid - 1;
        }
        return static_cast<unsigned short>(runs[lo].z + (e - runs[lo].x));
    };
    for (int e = t; e < 512; e += 256) {
        const int l = e >> 4, j = e & 15;
        unsigned short out = 0xFFFF;
        if (j < w) {
            const int col = cols[base + static_cast<int64_t>(j) * 32 + l];
            if (col >= 0) out = local(col);
        }
        lcol[c * 512 + e] = out;
    }
    if (t < 32) {
        const int64_t r = c * 32 + t;
        lown[c * 32 + t] = r < rows ? local(static_cast<int>(r + halo_lo)) : 0xFFFF;
    }
}

#endif  // CFD_EXPERIMENTAL

template <class M>
__global__ void sell_fill_kernel(const int64_t* __restrict__ offs, const int64_t* __restrict__ gcols,
                                 const M* __restrict__ gvals, int64_t rows,
                                 const int64_t* __restrict__ chunk_ptr, int* __restrict__ cols,
                                 M* __restrict__ vals, ColMap cm, int* __restrict__ err,
                                 unsigned long long* __restrict__ band) {
    const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t nch = (rows + kChunk - 1) / kChunk;
    if (r >= nch * kChunk) return;
    const int64_t chunk = r / kChunk;
    const int lane = static_cast<int>(r % kChunk);
    const int64_t base = chunk_ptr[chunk];
    const int64_t width = (chunk_ptr[chunk + 1] - base) / kChunk;
    const int64_t b = r < rows ? offs[r] : 0, e = r < rows ? offs[r + 1] : 0;
    int64_t dist = 0;
    for (int64_t j = 0; j < width; ++j) {
        const int64_t slot = base + j * kChunk + lane;
        if (b + j < e) {
            const int c = static_cast<int>(cm.map(gcols[b + j]));
            if (c < 0) atomicExch(err, 1);
            const int64_t d = c - (r + cm.halo_lo);
            dist = max(dist, d < 0 ? -d : d);
            cols[slot] = c;
            vals[slot] = gvals[b + j];
        } else {
            cols[slot] = -1;
            vals[slot] = M{};
        }
    }
    if (dist > 0) atomicMax(band, static_cast<unsigned long long>(dist));
}

}  // namespace

int step_slab_count(const Context& ctx, const StepArgs& s) {
    const int units = static_cast<int>(s.a->kind == CHEBFD_COMPLEX128 ? s.width_cols
                                       : (s.width_cols % 2 == 0 ? s.width_cols / 2 : s.width_cols));
    const TmaShape shape = tma_shape(ctx, units, s.row1 - s.row0);
    const int slab = ctx.slab_units > 0 ? std::min(ctx.slab_units, shape.slab_max) : shape.slab_max;
    return (units + slab - 1) / slab;
}

// width (columns) -> units per row / unit type; the instantiations live in
// step_c.cu (complex), step_r2.cu (real, two columns per 16-byte unit) and
// step_r1.cu (real, odd widths)
void launch_step(Context& ctx, const StepArgs& s, cudaStream_t st) {
    const int kind = s.a->kind;
    const int64_t width = s.width_cols;
    // the row-group kernel where the grouped form applies, else the SELL kernels
    if (kind == CHEBFD_COMPLEX128) {
        if (launch_ring_c(ctx, s, st, static_cast<int>(width), static_cast<int>(width))) return;
        if (!launch_group_c(ctx, s, st, static_cast<int>(width), static_cast<int>(width)))
            launch_step_c(ctx, s, st, static_cast<int>(width), static_cast<int>(width));
    } else if (width % 2 == 0) {
        if (!launch_group_r2(ctx, s, st, static_cast<int>(width / 2), static_cast<int>(width / 2)))
            launch_step_r2(ctx, s, st, static_cast<int>(width / 2), static_cast<int>(width / 2));
    } else {
        if (!launch_group_r1(ctx, s, st, static_cast<int>(width), static_cast<int>(width)))
            launch_step_r1(ctx, s, st, static_cast<int>(width), static_cast<int>(width));
    }
}

void ensure_scaled_grouped(Context& ctx, Matrix& a, double s, cudaStream_t st);  // group.cu

void ensure_scaled_values(Context& ctx, Matrix& a, double s, cudaStream_t st) {
    ensure_scaled_grouped(ctx, a, s, st);
    if (find_scaled(a, s)) return;
    if (a.scaled.size() >= 4) {
        // graphs may reference the evicted copy: the caller purges them
        a.scaled.erase(a.scaled.begin());
        a.scaled_evicted = true;
    }
    const int64_t n = std::max<int64_t>(a.entries, 1) * (a.kind ? 2 : 1);
    auto buf = std::make_unique<DeviceBuffer>(sizeof(double) * n);
    const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, ctx.num_sms * 8));
    scale_values_kernel<<<grid, 256, 0, st>>>(buf->as<double>(), a.vals.as<double>(), n, s);
    CFD_CUDA(cudaGetLastError());
    a.scaled.emplace_back(s, std::move(buf));
}

void launch_axpy(Context& ctx, Block& x, const Block& u, const Block& w, double c0, double c1,
                 double c2, cudaStream_t st) {
    const int64_t n = x.rows * x.width * (x.kind ? 2 : 1);
    if (n == 0) return;
    const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, ctx.num_sms * 8));
    axpy_kernel<<<grid, 256, 0, st>>>(static_cast<double*>(x.owned()),
                                      static_cast<const double*>(u.owned()),
                                      static_cast<const double*>(w.owned()), n, c0, c1, c2);
    CFD_CUDA(cudaGetLastError());
    ctx.launches++;
}

namespace {
template <bool CPLX, class T, int MODE>
void run_colreduce(Context& ctx, const Block& x, const Block& y, const double* lam, void* out,
                   cudaStream_t st, int units) {
    auto kernel = colreduce_kernel<CPLX, T, MODE>;
    for (int u0 = 0; u0 < units; u0 += 256) {
        const int us = std::min(256, units - u0);
        Geometry g = geometry(us);
        const size_t smem = static_cast<size_t>(g.threads) * sizeof(T);
        const int maxb = max_blocks_for(kernel, g.threads, smem, ctx.num_sms);
        const int64_t need = (x.rows + g.R - 1) / g.R;
        const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, maxb)));
        ctx.partials.ensure(
            std::max<size_t>(static_cast<size_t>(reduce_rows_needed(grid)) * us * sizeof(T), 1 << 20));
        ctx.counter.ensure(4096);
        kernel<<<grid, g.threads, smem, st>>>(
            static_cast<const T*>(x.owned()), static_cast<const T*>(y.owned()), lam, x.rows,
            units, u0, us, g.R, out, ctx.partials.as<T>(), ctx.counter.as<unsigned>());
        CFD_CUDA(cudaGetLastError());
        ctx.launches++;
    }
}
}  // namespace

void launch_column_reduce(Context& ctx, const Block& x, const Block& y, int mode, void* dev_out,
                          cudaStream_t st) {
    (void)mode;
    if (x.kind == CHEBFD_COMPLEX128)
        run_colreduce<true, double2, 0>(ctx, x, y, nullptr, dev_out, st, static_cast<int>(x.width));
    else if (x.width % 2 == 0)
        run_colreduce<false, double2, 0>(ctx, x, y, nullptr, dev_out, st, static_cast<int>(x.width / 2));
    else
        run_colreduce<false, double, 0>(ctx, x, y, nullptr, dev_out, st, static_cast<int>(x.width));
}

void launch_residual_sq(Context& ctx, const Block& av, const Block& v, const double* lam,
                        void* dev_out, cudaStream_t st) {
    if (av.kind == CHEBFD_COMPLEX128)
        run_colreduce<true, double2, 1>(ctx, av, v, lam, dev_out, st, static_cast<int>(av.width));
    else if (av.width % 2 == 0)
        run_colreduce<false, double2, 1>(ctx, av, v, lam, dev_out, st, static_cast<int>(av.width / 2));
    else
        run_colreduce<false, double, 1>(ctx, av, v, lam, dev_out, st, static_cast<int>(av.width));
}

void launch_axpy_scalar(Context& ctx, Block& w, const Block& q, double hr, double hi,
                        cudaStream_t st) {
    const int64_t n = w.rows * w.width;
    if (n == 0) return;
    const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, ctx.num_sms * 8));
    axpy_scalar_kernel<<<grid, 256, 0, st>>>(static_cast<double*>(w.owned()),
                                             static_cast<const double*>(q.owned()), n, w.kind, hr,
                                             hi);
    CFD_CUDA(cudaGetLastError());
    ctx.launches++;
}

void launch_scale_columns(Context& ctx, Block& b, const double* d_dev, cudaStream_t st) {
    const int64_t n = b.rows * b.width * (b.kind ? 2 : 1);
    if (n == 0) return;
    const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, ctx.num_sms * 8));
    divcols_kernel<<<grid, 256, 0, st>>>(static_cast<double*>(b.owned()), b.rows, b.width, b.kind,
                                         d_dev);
    CFD_CUDA(cudaGetLastError());
    ctx.launches++;
}

void launch_gather_rows(Context& ctx, void* dst, const void* src, const int64_t* idx, int64_t n,
                        int64_t row_bytes, cudaStream_t st) {
    if (n == 0 || row_bytes == 0) return;
    const int64_t tot = n * row_bytes / 8;
    const int grid = static_cast<int>(std::min<int64_t>((tot + 255) / 256, ctx.num_sms * 8));
    if (row_bytes % 16 == 0)
        gather_rows2_kernel<<<grid, 256, 0, st>>>(static_cast<double2*>(dst),
                                                  static_cast<const double2*>(src), idx, n,
                                                  row_bytes / 16);
    else
        gather_rows_kernel<<<grid, 256, 0, st>>>(static_cast<double*>(dst),
                                                 static_cast<const double*>(src), idx, n,
                                                 row_bytes / 8);
    CFD_CUDA(cudaGetLastError());
    ctx.launches++;
}

void launch_copy_columns(Context& ctx, Block& dst, int64_t d0, const Block& src, int64_t s0,
                         int64_t n, cudaStream_t st) {
    const int f = dst.kind ? 2 : 1;
    const int64_t tot = dst.rows * n * f;
    if (tot == 0) return;
    const int grid = static_cast<int>(std::min<int64_t>((tot + 255) / 256, ctx.num_sms * 8));
    copycols_kernel<<<grid, 256, 0, st>>>(static_cast<double*>(dst.owned()), dst.width * f, d0 * f,
                                          static_cast<const double*>(src.owned()), src.width * f,
                                          s0 * f, dst.rows, n * f);
    CFD_CUDA(cudaGetLastError());
    ctx.launches++;
}

void launch_philox_normal(Context& ctx, Block& b, uint64_t seed, cudaStream_t st) {
    const int64_t n = b.rows * b.width * (b.kind ? 2 : 1);
    if (n == 0) return;
    const int grid = ctx.num_sms * 4;
    // offset the Philox subsequence by the global first row so ranks differ
    philox_normal_kernel<<<grid, 256, 0, st>>>(static_cast<double*>(b.owned()), n,
                                               seed ^ (0x9E3779B97F4A7C15ULL * (b.row_begin + 1)));
    CFD_CUDA(cudaGetLastError());
    ctx.launches++;
}

void build_sell(Context& ctx, Matrix& m, const int64_t* d_offs, const int64_t* d_cols,
                const void* d_vals, cudaStream_t st) {
    const int64_t rows = m.part.local;
    m.nchunks = (rows + kChunk - 1) / kChunk;
    m.chunk_ptr.ensure(sizeof(int64_t) * (m.nchunks + 1));
    DeviceBuffer slots(sizeof(int64_t) * (m.nchunks + 1));
    m.chunk_full.ensure(static_cast<size_t>(m.nchunks) + 16);
    DeviceBuffer dmax(sizeof(int) * 4);  // max row length, error flag, band (uint64)
    CFD_CUDA(cudaMemsetAsync(dmax.p, 0, sizeof(int) * 4, st));
    CFD_CUDA(cudaMemsetAsync(slots.p, 0, sizeof(int64_t) * (m.nchunks + 1), st));
    if (m.nchunks > 0) {
        sell_width_kernel<<<static_cast<unsigned>((m.nchunks + 255) / 256), 256, 0, st>>>(
            d_offs, rows, m.nchunks, slots.as<int64_t>(), dmax.as<int>(),
            m.chunk_full.as<unsigned char>());
        CFD_CUDA(cudaGetLastError());
    }
    size_t tmp_bytes = 0;
    CFD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, slots.as<int64_t>(),
                                           m.chunk_ptr.as<int64_t>(), m.nchunks + 1, st));
    DeviceBuffer tmp(std::max<size_t>(tmp_bytes, 16));
    CFD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, slots.as<int64_t>(),
                                           m.chunk_ptr.as<int64_t>(), m.nchunks + 1, st));
    int64_t entries = 0;
    int maxlen = 0;
    CFD_CUDA(cudaMemcpyAsync(&entries, m.chunk_ptr.as<int64_t>() + m.nchunks, sizeof(int64_t),
                             cudaMemcpyDeviceToHost, st));
    CFD_CUDA(cudaMemcpyAsync(&maxlen, dmax.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CFD_CUDA(cudaStreamSynchronize(st));
    m.entries = entries;
    m.max_row_len = maxlen;
    if (static_cast<int64_t>(m.part.ext_rows()) >= (1LL << 31))
        fail(CHEBFD_ERR_UNSUPPORTED, "extended row count exceeds int32 column indices");
    m.cols.ensure(sizeof(int) * std::max<int64_t>(entries, 1));
    m.vals.ensure((m.kind ? 16 : 8) * std::max<int64_t>(entries, 1));
    // compact halos: the host already mapped the columns to extended rows (identity map)
    const ColMap cm = m.part.compact ? ColMap{0, m.part.ext_rows(), 0, 0, 0, 0} : colmap_of(m.part);
    const int64_t threads = m.nchunks * kChunk;
    if (threads > 0) {
        const unsigned grid = static_cast<unsigned>((threads + 255) / 256);
        if (m.kind)
            sell_fill_kernel<double2><<<grid, 256, 0, st>>>(
                d_offs, d_cols, static_cast<const double2*>(d_vals), rows,
                m.chunk_ptr.as<int64_t>(), m.cols.as<int>(), m.vals.as<double2>(), cm,
                dmax.as<int>() + 1, reinterpret_cast<unsigned long long*>(dmax.as<int>() + 2));
        else
            sell_fill_kernel<double><<<grid, 256, 0, st>>>(
                d_offs, d_cols, static_cast<const double*>(d_vals), rows,
                m.chunk_ptr.as<int64_t>(), m.cols.as<int>(), m.vals.as<double>(), cm,
                dmax.as<int>() + 1, reinterpret_cast<unsigned long long*>(dmax.as<int>() + 2));
        CFD_CUDA(cudaGetLastError());
    }
    int err = 0;
    unsigned long long band = 0;
    CFD_CUDA(cudaMemcpyAsync(&err, dmax.as<int>() + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CFD_CUDA(cudaMemcpyAsync(&band, dmax.as<int>() + 2, sizeof(band), cudaMemcpyDeviceToHost, st));
    CFD_CUDA(cudaStreamSynchronize(st));
    if (err) fail(CHEBFD_ERR_UNSUPPORTED, "matrix column outside this rank's rows and halos");
    m.band = static_cast<int64_t>(band);
    build_grouped(ctx, m, d_offs, d_cols, d_vals, st);
    // pair kernel tickets + one completion counter per 1024-row group, zeroed once
    // (every launch leaves them zeroed)
    const size_t groups = static_cast<size_t>((m.nchunks + 31) / 32);
    m.pair_sync.ensure(sizeof(unsigned) * (2 + groups) + 16);
    CFD_CUDA(cudaMemsetAsync(m.pair_sync.p, 0, m.pair_sync.bytes, st));
#if CFD_EXPERIMENTAL
    // staged-gather plan (kernel variant 2): rows of width <= 16 only
    m.stage_max_rows = 0;
    if (m.nchunks > 0 && maxlen <= 16 && m.part.ext_rows() < (1LL << 31)) {
        m.stage_runs.ensure(sizeof(int4) * kStageRuns * static_cast<size_t>(m.nchunks));
        m.stage_meta.ensure(sizeof(int2) * static_cast<size_t>(m.nchunks));
        m.stage_lcol.ensure(sizeof(unsigned short) * 512 * static_cast<size_t>(m.nchunks));
        m.stage_lown.ensure(sizeof(unsigned short) * 32 * static_cast<size_t>(m.nchunks));
        DeviceBuffer flags(sizeof(int) * 2);
        CFD_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int) * 2, st));
        stage_plan_kernel<<<static_cast<unsigned>(m.nchunks), 256, 0, st>>>(
            m.chunk_ptr.as<int64_t>(), m.cols.as<int>(), rows, m.part.halo_lo,
            m.stage_runs.as<int4>(), m.stage_meta.as<int2>(), m.stage_lcol.as<unsigned short>(),
            m.stage_lown.as<unsigned short>(), flags.as<int>(), flags.as<int>() + 1);
        CFD_CUDA(cudaGetLastError());
        int h[2] = {0, 0};
        CFD_CUDA(cudaMemcpyAsync(h, flags.p, sizeof(h), cudaMemcpyDeviceToHost, st));
        CFD_CUDA(cudaStreamSynchronize(st));
        m.stage_max_rows = h[1] ? 0 : h[0];
    }
#endif  // CFD_EXPERIMENTAL
}

}  // namespace cfd
