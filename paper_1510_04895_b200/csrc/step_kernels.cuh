// Step kernels of the fused Chebyshev filter and their launchers (sm_100a).
// Included by the per-scalar-type translation units step_c.cu / step_r2.cu /
// step_r1.cu (compiled in parallel) and, for the launch-geometry helpers, by
// kernels.cu.  See kernels.cu for the design summary.
#pragma once
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

namespace cfd {

namespace {

template <bool CPLX, class T, int KIND, int DMODE, int MAXW>
__global__ void __launch_bounds__(256, 2) step_kernel(const StepParams p) {
    using O = Ops<CPLX, T>;
    using M = typename O::M;
    constexpr int NDOT = dots_of(DMODE);
    const int t = threadIdx.x;
    const int rr = t / p.US;
    const int u = t - rr * p.US;
    const int R = p.R;
    const T* __restrict__ in = static_cast<const T*>(p.in);
    T* __restrict__ W = static_cast<T*>(p.w);
    T* __restrict__ X = static_cast<T*>(p.x);
    T* __restrict__ X0 = static_cast<T*>(p.x0);
    const M* __restrict__ vals = static_cast<const M*>(p.vals);
    const int* __restrict__ cols = p.cols;
    double coeff = p.c0, c1 = p.c1, c2 = p.c2;
    if (kind_fused(KIND) && p.coeff_dev) coeff = p.coeff_dev[p.coeff_index];
    if ((KIND == kStepFusedX2 || KIND == kStepFusedX3) && p.coeff_dev) c1 = p.coeff_dev[p.coeff_index - 1];
    if (KIND == kStepFusedX3 && p.coeff_dev) c2 = p.coeff_dev[p.coeff_index - 2];
    if (KIND == kStepStart2 && p.coeff_dev) {
        coeff = p.coeff_dev[0];
        c1 = p.coeff_dev[1];
        c2 = p.coeff_dev[2];
    }

    T acc_d[NDOT > 0 ? NDOT : 1];
    T comp_d[NDOT > 0 ? NDOT : 1];
#pragma unroll
    for (int d = 0; d < (NDOT > 0 ? NDOT : 1); ++d) {
        acc_d[d] = O::zero();
        comp_d[d] = O::zero();
    }

    const int64_t nrows = p.row1 - p.row0;
    const int64_t col_off = p.u_off + u;
    for (int64_t rg = blockIdx.x; rg * R < nrows; rg += gridDim.x) {
        const int64_t rl = rg * R + rr;
        if (rl >= nrows) continue;
        const int64_t r = p.row0 + rl;  // owned row
        const int64_t own = r * p.pitch + col_off;
        // own-row streams first: independent of the gathers, so they overlap
        T wi{}, xi{}, x0v{};
        if constexpr (kind_reads_w(KIND)) wi = ld_stream(&W[own]);
        if constexpr (kind_reads_x(KIND)) xi = ld_stream(&X[own]);
        if constexpr (DMODE == 2 && KIND != kStepStart2) x0v = ld_stream(&X0[own]);
        const int64_t chunk = r >> 5;
        const int lane = static_cast<int>(r & 31);
        const int64_t base = __ldg(&p.chunk_ptr[chunk]);
        const int width = static_cast<int>((__ldg(&p.chunk_ptr[chunk + 1]) - base) >> 5);
        const T acc = gather_row<O, T, M, MAXW>(cols, vals, in, base, width, lane, p.pitch, col_off,
                                                p.alpha);
        const T ui = ldg(&in[(r + p.halo_lo) * p.pitch + col_off]);
        step_epilogue<O, T, KIND, DMODE>(acc, ui, wi, xi, x0v, own, W, X, X0, p.beta, coeff, c1, c2,
                                         acc_d, comp_d);
    }

    if constexpr (NDOT > 0) {
        T acc_out[NDOT];
#pragma unroll
        for (int d = 0; d < NDOT; ++d) acc_out[d] = acc_d[d];
        const int US = p.US;
        const int uoff = p.u_off;
        void* outp = p.dots_out;
        const int64_t stride = p.dots_row_stride;
        grid_reduce<T, NDOT>(acc_out, R, US, static_cast<T*>(p.partials), p.part_base + blockIdx.x,
                             p.nparts, p.final_launch != 0, p.counter,
                             [&](int d, int uu, T v) {
                                 if (DMODE == 1)
                                     O::store_full(static_cast<T*>(outp), uoff + uu, v);
                                 else
                                     O::store_re(static_cast<double*>(outp) + d * stride,
                                                 uoff + uu, v);
                             });
    }
}

// ---- TMA-staged step kernel (default) ----------------------------------------------------
// A CTA walks over tiles of TR = max(32, R) rows (whole SELL chunks).  The
// tile's column indices and values -- contiguous in SELL -- are brought into
// shared memory by two TMA bulk copies (cp.async.bulk + mbarrier tx count),
// double-buffered so tile k+1 streams in while tile k is processed.  Threads
// read indices/values from shared memory, so registers only hold the
// gathered neighbour units in flight.  Own-row streams (W, X, x0) are plain
// coalesced loads issued ahead of the gathers.

// ORDER 0: persistent CTA-strided grid, row order (any launch); ORDER 1: non-persistent
// grid of p.tile_a consecutive tiles per CTA in the band (2.5D) order (dot-free launches
// on lattice operators whose planes exceed the L2 budget; see set_band_order)
template <bool CPLX, class T, int KIND, int DMODE, int MAXW, int ORDER = 0>
__global__ void __launch_bounds__(CFD_TMA_THREADS, CFD_TMA_MINB) step_tma_kernel(const StepParams p) {
    using O = Ops<CPLX, T>;
    using M = typename O::M;
    constexpr int NDOT = dots_of(DMODE);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[2];
    const int t = threadIdx.x;
    const int US = p.US;
    const int rr = t / US;
    const int u = t - rr * US;
    const int R = p.R;
    const int TR = R > p.tr ? R : p.tr;  // rows per tile (whole chunks)
    const int NCH = TR / 32;
    const int cap = MAXW * TR;  // slots per buffer
    int* cols_s = reinterpret_cast<int*>(smem_raw);
    M* vals_s = reinterpret_cast<M*>(smem_raw + ((2 * cap * sizeof(int) + 15) & ~size_t(15)));
    // plain dot sums (modes 2-4) accumulate in shared memory, one slot per thread and
    // dot, so no accumulator register is live across a row's gathers (C2, two moment
    // dots per row: 734 us per step with complex register accumulators -- ptxas split
    // the eleven gathers into two batches --, 713 us with real-part registers, 685 us
    // here; no dots: 587 us)
    constexpr bool SACC = NDOT > 0 && DMODE != 1;
    auto* sacc = reinterpret_cast<std::conditional_t<DMODE == 1, T, typename O::DT>*>(
        smem_raw + ((((2 * cap * sizeof(int) + 15) & ~size_t(15)) + 2 * cap * sizeof(M) + 15) & ~size_t(15)));

    const int cu = p.u_off + u;
    const T* __restrict__ inu = static_cast<const T*>(p.in) + cu;
    T* __restrict__ W = static_cast<T*>(p.w) + cu;
    T* __restrict__ X = static_cast<T*>(p.x) + cu;
    T* __restrict__ X0 = static_cast<T*>(p.x0) + cu;
    const M* __restrict__ gvals = static_cast<const M*>(p.svals);  // pre-multiplied by alpha
    const int pitch = p.pitch;
    const int64_t halo = p.halo_lo;
    double coeff = p.c0, c1 = p.c1, c2 = p.c2;
    if (kind_fused(KIND) && p.coeff_dev) coeff = p.coeff_dev[p.coeff_index];
    if ((KIND == kStepFusedX2 || KIND == kStepFusedX3) && p.coeff_dev) c1 = p.coeff_dev[p.coeff_index - 1];
    if (KIND == kStepFusedX3 && p.coeff_dev) c2 = p.coeff_dev[p.coeff_index - 2];
    if (KIND == kStepStart2 && p.coeff_dev) {
        coeff = p.coeff_dev[0];
        c1 = p.coeff_dev[1];
        c2 = p.coeff_dev[2];
    }
    // dot accumulators: Kahan <x, w> (mode 1) keeps complex units; moments and plain
    // dots only need real parts (O::DT)
    using A = std::conditional_t<DMODE == 1, T, typename O::DT>;
    A acc_d[NDOT > 0 ? NDOT : 1];
    A comp_d[NDOT > 0 ? NDOT : 1];
#pragma unroll
    for (int d = 0; d < (NDOT > 0 ? NDOT : 1); ++d) {
        acc_d[d] = A{};
        comp_d[d] = A{};
    }

#if CFD_L2_HINTS
    const uint64_t pol_keep = l2_make_policy(1);
    const uint64_t pol_stream = l2_make_policy(2);
#endif
    const int64_t row0 = p.row0, row1 = p.row1;
    const int64_t cbeg = row0 >> 5;
    const int64_t cend = (row1 + 31) >> 5;
    const int64_t ntiles = row1 > row0 ? (cend - cbeg + NCH - 1) / NCH : 0;
    const int64_t* __restrict__ cptr = p.chunk_ptr;

    auto first_chunk = [&](int64_t tile) -> int64_t {
        if constexpr (ORDER == 0)
            return cbeg + tile * NCH;
        else
            return tile_first_chunk(p, tile, cbeg, NCH);
    };
    auto issue = [&](int64_t tile, int buf) {
        const int64_t c0 = first_chunk(tile);
        const int64_t c1e = min(c0 + NCH, cend);
        const int64_t s0 = cptr[c0], s1 = cptr[c1e];
        const unsigned n = static_cast<unsigned>(s1 - s0);
        const unsigned bc = n * 4u, bv = n * static_cast<unsigned>(sizeof(M));
        mbar_arrive_expect_tx(&bars[buf], bc + bv);
        if (n) {
            tma_load_1d(cols_s + buf * cap, p.cols + s0, bc, &bars[buf]);
            tma_load_1d(vals_s + buf * cap, gvals + s0, bv, &bars[buf]);
        }
    };

    // one row of the current tile; FAST: every chunk of the tile is full with
    // width MAXW (no padding predicates, slot offsets computed, not loaded)
    // (lr: r relative to the tile's first row c0 * 32)
    auto row = [&](auto fast_tag, int lr, int64_t c0, int64_t sbase, const int* cs, const M* vs) {
        constexpr bool FAST = decltype(fast_tag)::value;
        const int64_t r = c0 * 32 + lr;
        const int lane = lr & 31;
        int coff, w;
        if constexpr (FAST) {
            coff = (lr >> 5) * (32 * MAXW) + lane;
            w = MAXW;
        } else {
            const int64_t chunk = r >> 5;
            const int64_t cb = __ldg(&cptr[chunk]);
            coff = static_cast<int>(cb - sbase) + lane;
            w = static_cast<int>((__ldg(&cptr[chunk + 1]) - cb) >> 5);
        }
        const int64_t own = r * pitch;
        T wi{}, xi{}, x0v{};
#if CFD_L2_HINTS
        // the z +- 1 plane reuse of gathered rows survives the streams
        auto ldg = [&](const T* q) { return ldg_pol(q, pol_keep); };
        auto ld_stream = [&](const T* q) { return lds_pol(q, pol_stream); };
#endif
        if constexpr (kind_reads_w(KIND)) wi = ld_stream(&W[own]);
        if constexpr (kind_reads_x(KIND)) xi = ld_stream(&X[own]);
        if constexpr (DMODE == 2 && KIND != kStepStart2) x0v = ld_stream(&X0[own]);
        T acc = O::zero();
        if constexpr (FAST) {
            int c[MAXW];
#pragma unroll
            for (int j = 0; j < MAXW; ++j) c[j] = cs[coff + j * 32];
            T g[MAXW];
#pragma unroll
            for (int j = 0; j < MAXW; ++j) g[j] = ldg(&inu[static_cast<int64_t>(c[j]) * pitch]);
#pragma unroll
            for (int j = 0; j < MAXW; ++j) acc = O::vadd(acc, O::prod(vs[coff + j * 32], g[j]));
        } else {
            int c[MAXW];
#pragma unroll
            for (int j = 0; j < MAXW; ++j) c[j] = (j < w) ? cs[coff + j * 32] : -1;
            T g[MAXW];
#pragma unroll
            for (int j = 0; j < MAXW; ++j)
                if (c[j] >= 0) g[j] = ldg(&inu[static_cast<int64_t>(c[j]) * pitch]);
#pragma unroll
            for (int j = 0; j < MAXW; ++j)
                if (c[j] >= 0) acc = O::vadd(acc, O::prod(vs[coff + j * 32], g[j]));
        }
        const T ui = ldg(&inu[(r + halo) * pitch]);
        if constexpr (SACC) {
            A dl[NDOT], dc[NDOT];
#pragma unroll
            for (int d = 0; d < NDOT; ++d) dl[d] = dc[d] = A{};
            step_epilogue<O, T, KIND, DMODE>(acc, ui, wi, xi, x0v, own, W, X, X0, p.beta, coeff, c1,
                                             c2, dl, dc);
            // 0 + v is exact: the same roundings as accumulating in a register
#pragma unroll
            for (int d = 0; d < NDOT; ++d) sacc[d * blockDim.x + t] = tadd(sacc[d * blockDim.x + t], dl[d]);
        } else {
            step_epilogue<O, T, KIND, DMODE>(acc, ui, wi, xi, x0v, own, W, X, X0, p.beta, coeff, c1,
                                             c2, acc_d, comp_d);
        }
    };

    // two rows per thread, all 2 x MAXW gathers issued together (V_n-only steps without
    // dots: no X / x0 / accumulator registers, so the second row's gathers fit the register
    // budget; ptxas still interleaves part of them): C2 496 -> 473 us per V_n-only step.
    // Rows it + rr and it + R + rr of the tile (needs TR >= 2R).
    // lra, lrb: rows relative to the tile's first row c0 * 32 (slot offsets need no c0)
    auto row2 = [&](int lra, int lrb, int64_t c0, const int* cs, const M* vs) {
        const int64_t ra = c0 * 32 + lra, rb = c0 * 32 + lrb;
#if CFD_L2_HINTS
        auto ldg = [&](const T* q) { return ldg_pol(q, pol_keep); };
        auto ld_stream = [&](const T* q) { return lds_pol(q, pol_stream); };
#endif
        const int coffa = (lra >> 5) * (32 * MAXW) + (lra & 31);
        const int coffb = (lrb >> 5) * (32 * MAXW) + (lrb & 31);
        const int64_t owna = ra * pitch, ownb = rb * pitch;
        const T wia = ld_stream(&W[owna]);
        const T wib = ld_stream(&W[ownb]);
        T ga[MAXW], gb[MAXW];
#pragma unroll
        for (int j = 0; j < MAXW; ++j) ga[j] = ldg(&inu[static_cast<int64_t>(cs[coffa + j * 32]) * pitch]);
#pragma unroll
        for (int j = 0; j < MAXW; ++j) gb[j] = ldg(&inu[static_cast<int64_t>(cs[coffb + j * 32]) * pitch]);
        T acca = O::zero(), accb = O::zero();
#pragma unroll
        for (int j = 0; j < MAXW; ++j) acca = O::vadd(acca, O::prod(vs[coffa + j * 32], ga[j]));
#pragma unroll
        for (int j = 0; j < MAXW; ++j) accb = O::vadd(accb, O::prod(vs[coffb + j * 32], gb[j]));
        const T uia = ldg(&inu[(ra + halo) * pitch]);
        const T uib = ldg(&inu[(rb + halo) * pitch]);
        // kernels.hpp:142: w' = tmp + 2b u_i - w_i
        st_stream(&W[owna], O::vsub(O::vadd(acca, O::smul(p.beta, uia)), wia));
        st_stream(&W[ownb], O::vsub(O::vadd(accb, O::smul(p.beta, uib)), wib));
    };
    constexpr bool TWO_ROWS = KIND == kStepRecur && DMODE == 0 && MAXW >= 8;
    const bool two_rows = TWO_ROWS && TR >= 2 * R && TR % (2 * R) == 0;

    if constexpr (SACC) {
#pragma unroll
        for (int d = 0; d < NDOT; ++d) sacc[d * blockDim.x + t] = A{};
    }
    if (t == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    // Tile schedule.  ORDER 0: CTA b takes tiles b, b + grid, ... (a fixed CTA-to-tile map:
    // per-CTA dot partials, hence the reduced dots, are bitwise reproducible).  ORDER 1:
    // tiles b * tile_a + k, k < tile_a, of a non-persistent grid: the block scheduler hands
    // out CTAs in order, so the wavefront stays compact (persistent CTAs drift apart by
    // hundreds of MB of rows, which defeats the band order's L2 reuse).
    const int64_t tstride = ORDER == 0 ? static_cast<int64_t>(gridDim.x) : 1;
    int64_t tile = ORDER == 0 ? static_cast<int64_t>(blockIdx.x) : blockIdx.x * p.tile_a;
    const int64_t tend = ORDER == 0 ? ntiles : min(ntiles, tile + p.tile_a);
    // programmatic dependent launch: the launch and the set-up above overlap the previous
    // kernel's tail; nothing in global memory is read before that grid has completed and
    // flushed (its output may be this step's operand, or freshly scaled matrix values).
    // A no-op when launched without the PDL attribute.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (t == 0 && tile < tend) issue(tile, 0);
    unsigned phases = 0u;  // bit b = parity of buffer b's next completion
    for (int k = 0; tile < tend; ++k, tile += tstride) {
        const int buf = k & 1;
        if (tile + tstride >= tend) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        if (t == 0 && tile + tstride < tend) issue(tile + tstride, buf ^ 1);
        const int64_t c0 = first_chunk(tile);
        const int64_t c1e = min(c0 + NCH, cend);
        const int64_t sbase = cptr[c0];
        // fast tile: all chunks full, width == MAXW, tile fully inside [row0, row1)
        bool fast = (cptr[c1e] - sbase) == (c1e - c0) * 32 * MAXW && c0 * 32 >= row0 &&
                    c1e * 32 <= row1 && (c1e - c0) == NCH;
        for (int64_t c = c0; fast && c < c1e; ++c) fast = __ldg(&p.chunk_full[c]) != 0;
        mbar_wait(&bars[buf], (phases >> buf) & 1u);
        phases ^= 1u << buf;
        const int* cs = cols_s + buf * cap;
        const M* vs = vals_s + buf * cap;
        if (fast) {
            if (two_rows) {
                for (int it = 0; it < TR; it += 2 * R)
                    row2(it + rr, it + R + rr, c0, cs, vs);
            } else {
                for (int it = 0; it < TR; it += R)
                    row(std::true_type{}, it + rr, c0, sbase, cs, vs);
            }
        } else {
            for (int it = 0; it < TR; it += R) {
                const int64_t r = c0 * 32 + it + rr;
                if (r < row0 || r >= row1) continue;
                row(std::false_type{}, it + rr, c0, sbase, cs, vs);
            }
        }
        __syncthreads();  // buffer `buf` is refilled two tiles later
    }

    if constexpr (NDOT > 0) {
        A acc_out[NDOT];
#pragma unroll
        for (int d = 0; d < NDOT; ++d) acc_out[d] = SACC ? sacc[d * blockDim.x + t] : acc_d[d];
        __syncthreads();  // grid_reduce reuses the shared memory
        const int uoff = p.u_off;
        void* outp = p.dots_out;
        const int64_t dstride = p.dots_row_stride;
        grid_reduce<A, NDOT>(acc_out, R, US, static_cast<A*>(p.partials), p.part_base + blockIdx.x,
                             p.nparts, p.final_launch != 0, p.counter,
                             [&](int d, int uu, A vv) {
                                 if constexpr (DMODE == 1)
                                     O::store_full(static_cast<T*>(outp), uoff + uu, vv);
                                 else
                                     O::store_re(static_cast<double*>(outp) + d * dstride,
                                                 uoff + uu, vv);
                             });
    }
}

// ---- two units per thread, 256-bit accesses, W / X staged by TMA (default where it applies) ----
// Same arithmetic and order as step_tma_kernel, but each thread owns two
// adjacent 16-byte units of its row: the eleven gathers are LDG.256 (32 B per
// thread, 512 B per half warp), so a row in flight costs half the threads; the
// own-row streams W / X (/ x0) of the tile come into shared memory by one TMA
// bulk copy each with the matrix chunk, so no register holds them while the
// gathers are in flight.  Net: about twice the rows in flight per SM at the
// same register budget (the TMA kernel's limit), and half the load instructions.
template <class T>
struct alignas(32) U2 {
    T a, b;
};
template <>
__device__ __forceinline__ U2<double2> tadd<U2<double2>>(U2<double2> x, U2<double2> y) {
    return {tadd(x.a, y.a), tadd(x.b, y.b)};
}
__device__ __forceinline__ U2<double2> ld256_nc(const double2* p) {
    U2<double2> v;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v.a.x), "=d"(v.a.y), "=d"(v.b.x), "=d"(v.b.y)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st256_cs(double2* p, const U2<double2>& v) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.a.x), "d"(v.a.y),
                 "d"(v.b.x), "d"(v.b.y)
                 : "memory");
}

// the per-unit epilogue of step_epilogue, on values already in registers,
// returning what step_epilogue stores (so the two units store as one 256-bit op)
template <class O, class T, int KIND, int DMODE, int NA>
__device__ __forceinline__ void epilogue2(const T acc, const T ui, const T wi, const T xi,
                                          const T x0v, T& w_out, T& x_out, T& x0_out, double beta,
                                          double coeff, double c1, double c2, T (&acc_d)[NA],
                                          T (&comp_d)[NA]) {
    if constexpr (KIND == kStepSpmmvm) {
        T y = acc;
        if (beta != 0.0) y = O::vadd(y, O::smul(beta, ui));  // kernels.hpp:62-65
        w_out = y;
        if constexpr (DMODE == 3 || DMODE == 4) {
            x0_out = ui;
            acc_d[0] = O::vadd(acc_d[0], O::cdot(ui, ui));
            acc_d[1] = O::vadd(acc_d[1], O::cdot(ui, y));
        }
    } else if constexpr (KIND == kStepStart2) {
        T wr = acc;
        if (beta != 0.0) wr = O::vadd(wr, O::smul(beta, ui));
        const T wn = O::vadd(O::vadd(O::smul(1.0, wr), O::smul(-1.0, xi)), O::smul(0.0, xi));
        w_out = wn;
        if constexpr (DMODE == 2) acc_d[0] = O::vadd(acc_d[0], O::cdot(xi, wn));
        if constexpr (DMODE == 4) moment_pair<O>(acc_d, ui, wn);
        x_out = O::vadd(O::vadd(O::smul(coeff, xi), O::smul(c1, ui)), O::smul(c2, wn));
    } else {
        const T wn = O::vsub(O::vadd(acc, O::smul(beta, ui)), wi);
        w_out = wn;
        if constexpr (KIND == kStepFused) {
            if constexpr (DMODE == 1) kahan_add<T>(acc_d[0], comp_d[0], O::cdot(xi, wn));
            if constexpr (DMODE == 2) acc_d[0] = O::vadd(acc_d[0], O::cdot(x0v, wn));
            x_out = O::vadd(xi, O::smul(coeff, wn));
        } else if constexpr (KIND == kStepFusedX2) {
            if constexpr (DMODE == 2) acc_d[0] = O::vadd(acc_d[0], O::cdot(x0v, wn));
            x_out = O::vadd(O::vadd(xi, O::smul(c1, ui)), O::smul(coeff, wn));
        } else if constexpr (KIND == kStepFusedX3) {
            if constexpr (DMODE == 2) acc_d[0] = O::vadd(acc_d[0], O::cdot(x0v, wn));
            x_out = O::vadd(O::vadd(O::vadd(xi, O::smul(c2, wi)), O::smul(c1, ui)), O::smul(coeff, wn));
        } else {
            if constexpr (DMODE == 2) acc_d[0] = O::vadd(acc_d[0], O::cdot(x0v, wn));
        }
        if constexpr (DMODE == 4) moment_pair<O>(acc_d, ui, wn);
        if constexpr (DMODE == 5) moment_quad<O>(acc_d, wi, ui, wn);
        if constexpr (DMODE == 6) {
            acc_d[0] = O::vadd(acc_d[0], O::cdot(ui, wn));
            acc_d[1] = O::vadd(acc_d[1], O::cdot(wn, wn));
        }
    }
}

template <bool CPLX, int KIND, int DMODE, int MAXW>
__global__ void __launch_bounds__(256, 2) step_tma2_kernel(const StepParams p) {
    using T = double2;
    using O = Ops<CPLX, T>;
    using M = typename O::M;
    using P = U2<T>;
    constexpr int NDOT = dots_of(DMODE);
    constexpr bool HAS_W = kind_reads_w(KIND);
    constexpr bool HAS_X = kind_reads_x(KIND);
    constexpr bool HAS_X0 = (DMODE == 2 && KIND != kStepStart2);
    constexpr int NS = (HAS_W ? 1 : 0) + (HAS_X ? 1 : 0) + (HAS_X0 ? 1 : 0);  // staged streams
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[2];
    const int t = threadIdx.x;
    const int HS = p.US >> 1;  // threads per row
    const int rr = t / HS;
    const int u2 = t - rr * HS;
    const int R = p.R;          // rows per pass
    constexpr int TR = 32;      // one chunk per tile
    const int pitch = p.pitch;  // == p.US (whole rows)
    const int cap = MAXW * TR;
    const size_t sell_bytes = ((cap * sizeof(int) + 15) & ~size_t(15)) + cap * sizeof(M);
    const size_t row_tile = static_cast<size_t>(TR) * pitch * sizeof(T);
    const size_t stage_bytes = sell_bytes + NS * row_tile;
    auto cols_s = [&](int b) { return reinterpret_cast<const int*>(smem_raw + b * stage_bytes); };
    auto vals_s = [&](int b) {
        return reinterpret_cast<const M*>(smem_raw + b * stage_bytes +
                                          ((cap * sizeof(int) + 15) & ~size_t(15)));
    };
    auto rows_s = [&](int b, int k) {
        return reinterpret_cast<const T*>(smem_raw + b * stage_bytes + sell_bytes + k * row_tile);
    };

    const int cu = 2 * u2;
    const T* __restrict__ inu = static_cast<const T*>(p.in) + cu;
    T* __restrict__ W = static_cast<T*>(p.w);
    T* __restrict__ X = static_cast<T*>(p.x);
    T* __restrict__ X0 = static_cast<T*>(p.x0);
    const M* __restrict__ gvals = static_cast<const M*>(p.svals);
    const int64_t halo = p.halo_lo;
    double coeff = p.c0, c1 = p.c1, c2 = p.c2;
    if (kind_fused(KIND) && p.coeff_dev) coeff = p.coeff_dev[p.coeff_index];
    if ((KIND == kStepFusedX2 || KIND == kStepFusedX3) && p.coeff_dev) c1 = p.coeff_dev[p.coeff_index - 1];
    if (KIND == kStepFusedX3 && p.coeff_dev) c2 = p.coeff_dev[p.coeff_index - 2];
    if (KIND == kStepStart2 && p.coeff_dev) {
        coeff = p.coeff_dev[0];
        c1 = p.coeff_dev[1];
        c2 = p.coeff_dev[2];
    }
    P acc_d[NDOT > 0 ? NDOT : 1];
    P comp_d[NDOT > 0 ? NDOT : 1];
#pragma unroll
    for (int d = 0; d < (NDOT > 0 ? NDOT : 1); ++d) {
        acc_d[d] = P{O::zero(), O::zero()};
        comp_d[d] = P{O::zero(), O::zero()};
    }
    const int64_t row0 = p.row0, row1 = p.row1;
    const int64_t cbeg = row0 >> 5;
    const int64_t ntiles = row1 > row0 ? ((row1 + 31) >> 5) - cbeg : 0;
    const int64_t* __restrict__ cptr = p.chunk_ptr;

    auto issue = [&](int64_t tile, int b) {
        const int64_t c = cbeg + tile;
        const int64_t s0 = cptr[c], s1 = cptr[c + 1];
        const unsigned n = static_cast<unsigned>(s1 - s0);
        const int64_t ra = max(c * 32, row0), rb = min(c * 32 + 32, row1);
        const unsigned rows_b = static_cast<unsigned>((rb - ra) * pitch * sizeof(T));
        unsigned char* base = smem_raw + b * stage_bytes;
        mbar_arrive_expect_tx(&bars[b], n * 4u + n * static_cast<unsigned>(sizeof(M)) + NS * rows_b);
        if (n) {
            tma_load_1d(base, p.cols + s0, n * 4u, &bars[b]);
            tma_load_1d(base + ((cap * sizeof(int) + 15) & ~size_t(15)), gvals + s0,
                        n * static_cast<unsigned>(sizeof(M)), &bars[b]);
        }
        const size_t off = static_cast<size_t>(ra - c * 32) * pitch * sizeof(T);
        int k = 0;
        if constexpr (HAS_W) tma_load_1d(base + sell_bytes + (k++) * row_tile + off, W + ra * pitch, rows_b, &bars[b]);
        if constexpr (HAS_X) tma_load_1d(base + sell_bytes + (k++) * row_tile + off, X + ra * pitch, rows_b, &bars[b]);
        if constexpr (HAS_X0) tma_load_1d(base + sell_bytes + (k++) * row_tile + off, X0 + ra * pitch, rows_b, &bars[b]);
        (void)k;
    };

    auto row = [&](auto fast_tag, int64_t r, int64_t c, int64_t sbase, int b) {
        constexpr bool FAST = decltype(fast_tag)::value;
        const int* cs = cols_s(b);
        const M* vs = vals_s(b);
        const int lane = static_cast<int>(r & 31);
        int coff, w;
        if constexpr (FAST) {
            coff = lane;
            w = MAXW;
        } else {
            const int64_t cb = __ldg(&cptr[c]);
            coff = static_cast<int>(cb - sbase) + lane;
            w = static_cast<int>((__ldg(&cptr[c + 1]) - cb) >> 5);
        }
        P acc{O::zero(), O::zero()};
        int cc[MAXW];
#pragma unroll
        for (int j = 0; j < MAXW; ++j) cc[j] = (FAST || j < w) ? cs[coff + j * 32] : -1;
        P g[MAXW];
#pragma unroll
        for (int j = 0; j < MAXW; ++j)
            if (FAST || cc[j] >= 0) g[j] = ld256_nc(&inu[static_cast<int64_t>(cc[j]) * pitch]);
#pragma unroll
        for (int j = 0; j < MAXW; ++j)
            if (FAST || cc[j] >= 0) {
                const M v = vs[coff + j * 32];
                acc.a = O::vadd(acc.a, O::prod(v, g[j].a));
                acc.b = O::vadd(acc.b, O::prod(v, g[j].b));
            }
        const P ui = ld256_nc(&inu[(r + halo) * pitch]);
        const int lr = static_cast<int>(r - c * 32);
        P wi{}, xi{}, x0v{};
        int k = 0;
        if constexpr (HAS_W) wi = *reinterpret_cast<const P*>(rows_s(b, k++) + lr * pitch + cu);
        if constexpr (HAS_X) xi = *reinterpret_cast<const P*>(rows_s(b, k++) + lr * pitch + cu);
        if constexpr (HAS_X0) x0v = *reinterpret_cast<const P*>(rows_s(b, k++) + lr * pitch + cu);
        (void)k;
        P wo{}, xo{}, x0o{};
        T ad_a[NDOT > 0 ? NDOT : 1], cd_a[NDOT > 0 ? NDOT : 1], ad_b[NDOT > 0 ? NDOT : 1],
            cd_b[NDOT > 0 ? NDOT : 1];
#pragma unroll
        for (int d = 0; d < (NDOT > 0 ? NDOT : 1); ++d) {
            ad_a[d] = acc_d[d].a;
            cd_a[d] = comp_d[d].a;
            ad_b[d] = acc_d[d].b;
            cd_b[d] = comp_d[d].b;
        }
        epilogue2<O, T, KIND, DMODE>(acc.a, ui.a, wi.a, xi.a, x0v.a, wo.a, xo.a, x0o.a, p.beta,
                                     coeff, c1, c2, ad_a, cd_a);
        epilogue2<O, T, KIND, DMODE>(acc.b, ui.b, wi.b, xi.b, x0v.b, wo.b, xo.b, x0o.b, p.beta,
                                     coeff, c1, c2, ad_b, cd_b);
#pragma unroll
        for (int d = 0; d < (NDOT > 0 ? NDOT : 1); ++d) {
            acc_d[d] = P{ad_a[d], ad_b[d]};
            comp_d[d] = P{cd_a[d], cd_b[d]};
        }
        const int64_t own = r * pitch + cu;
        st256_cs(&W[own], wo);
        if constexpr (KIND == kStepSpmmvm && DMODE == 3) st256_cs(&X0[own], x0o);
        if constexpr (kind_reads_x(KIND)) st256_cs(&X[own], xo);
    };

    if (t == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    int64_t tile = blockIdx.x;
    // programmatic dependent launch: W / X tiles (TMA) are the previous step's output
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (t == 0 && tile < ntiles) issue(tile, 0);
    unsigned phases = 0u;
    for (int k = 0; tile < ntiles; ++k, tile += gridDim.x) {
        const int buf = k & 1;
        if (tile + gridDim.x >= ntiles) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        if (t == 0 && tile + gridDim.x < ntiles) issue(tile + gridDim.x, buf ^ 1);
        const int64_t c = cbeg + tile;
        const int64_t sbase = cptr[c];
        const bool fast = (cptr[c + 1] - sbase) == 32 * MAXW && c * 32 >= row0 && c * 32 + 32 <= row1 &&
                          __ldg(&p.chunk_full[c]) != 0;
        mbar_wait(&bars[buf], (phases >> buf) & 1u);
        phases ^= 1u << buf;
        if (fast) {
            for (int it = 0; it < TR; it += R) row(std::true_type{}, c * 32 + it + rr, c, sbase, buf);
        } else {
            for (int it = 0; it < TR; it += R) {
                const int64_t r = c * 32 + it + rr;
                if (r < row0 || r >= row1) continue;
                row(std::false_type{}, r, c, sbase, buf);
            }
        }
        __syncthreads();
    }

    if constexpr (NDOT > 0) {
        void* outp = p.dots_out;
        const int64_t dstride = p.dots_row_stride;
        grid_reduce<P, NDOT>(acc_d, R, HS, reinterpret_cast<P*>(p.partials), p.part_base + blockIdx.x,
                             p.nparts, p.final_launch != 0, p.counter, [&](int d, int uu, P vv) {
                                 if (DMODE == 1) {
                                     O::store_full(static_cast<T*>(outp), 2 * uu, vv.a);
                                     O::store_full(static_cast<T*>(outp), 2 * uu + 1, vv.b);
                                 } else {
                                     O::store_re(static_cast<double*>(outp) + d * dstride, 2 * uu, vv.a);
                                     O::store_re(static_cast<double*>(outp) + d * dstride, 2 * uu + 1, vv.b);
                                 }
                             });
    }
}

#if CFD_EXPERIMENTAL
// ---- staged-gather step kernel (kernel variant 2) -------------------------------------------
// One tile = one 32-row SELL chunk, one CTA per SM, two shared-memory stages.
// Warp 0 stages tile k+1 by TMA bulk copies -- the chunk's values, its plan
// (16-bit local column indices, row-major per row) and every run of gathered
// rows the chunk reads -- while the CTA computes tile k entirely from shared
// memory; W / X (/ x0) of tile k+1 are prefetched into registers.  No gather
// is in flight in registers, so the latency that bounds the TMA kernel's
// 16 warps/SM is replaced by bulk copies.  One warp = one row slot (32 units
// = 512 B: complex n_b = 32 or real n_b = 64); 8 warps x 4 rows per tile.
// Accumulation order per row = stored order: bit-identical to step_tma_kernel.
struct StagePlan {
    const int4* runs;
    const int2* meta;
    const unsigned short* lcol;
    const unsigned short* lown;
    int cap_rows;  // U rows per stage
    int nstage;    // shared-memory stages (2 or 3): tiles staged ahead = nstage - 1
};

template <bool CPLX, class T, int KIND, int DMODE, int MAXW>
__global__ void __launch_bounds__(256, 1) step_stage_kernel(const StepParams p, const StagePlan sp) {
    using O = Ops<CPLX, T>;
    using M = typename O::M;
    constexpr int US = 32, R = 8, NP = 4;
    constexpr int NDOT = dots_of(DMODE);
    constexpr bool HAS_W = kind_reads_w(KIND);
    constexpr bool HAS_X = kind_reads_x(KIND);
    constexpr bool HAS_X0 = (DMODE == 2 && KIND != kStepStart2);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[3];
    const int t = threadIdx.x;
    const int rr = t >> 5, u = t & 31;
    const int ns = sp.nstage;
    const size_t u_bytes = static_cast<size_t>(sp.cap_rows) * US * sizeof(T);
    const size_t v_bytes = 32 * MAXW * sizeof(M);
    const size_t stage_bytes = u_bytes + v_bytes + 32 * 16 * 2 + 32 * 2;
    auto U_s = [&](int b) { return reinterpret_cast<const T*>(smem_raw + b * stage_bytes); };
    auto V_s = [&](int b) { return reinterpret_cast<const M*>(smem_raw + b * stage_bytes + u_bytes); };
    auto LC_s = [&](int b) {
        return reinterpret_cast<const unsigned short*>(smem_raw + b * stage_bytes + u_bytes + v_bytes);
    };
    auto LO_s = [&](int b) {
        return reinterpret_cast<const unsigned short*>(smem_raw + b * stage_bytes + u_bytes + v_bytes +
                                                       1024);
    };

    const T* __restrict__ in = static_cast<const T*>(p.in);
    T* __restrict__ W = static_cast<T*>(p.w) + u;
    T* __restrict__ X = static_cast<T*>(p.x) + u;
    T* __restrict__ X0 = static_cast<T*>(p.x0) + u;
    const M* __restrict__ gvals = static_cast<const M*>(p.svals);
    const int pitch = p.pitch;
    double coeff = p.c0, c1 = p.c1, c2 = p.c2;
    if (kind_fused(KIND) && p.coeff_dev) coeff = p.coeff_dev[p.coeff_index];
    if ((KIND == kStepFusedX2 || KIND == kStepFusedX3) && p.coeff_dev) c1 = p.coeff_dev[p.coeff_index - 1];
    if (KIND == kStepFusedX3 && p.coeff_dev) c2 = p.coeff_dev[p.coeff_index - 2];
    if (KIND == kStepStart2 && p.coeff_dev) {
        coeff = p.coeff_dev[0];
        c1 = p.coeff_dev[1];
        c2 = p.coeff_dev[2];
    }
    T acc_d[NDOT > 0 ? NDOT : 1];
    T comp_d[NDOT > 0 ? NDOT : 1];
#pragma unroll
    for (int d = 0; d < (NDOT > 0 ? NDOT : 1); ++d) {
        acc_d[d] = O::zero();
        comp_d[d] = O::zero();
    }
    const int64_t row0 = p.row0, row1 = p.row1;
    const int64_t cbeg = row0 >> 5;
    const int64_t ntiles = row1 > row0 ? ((row1 + 31) >> 5) - cbeg : 0;
    const int64_t* __restrict__ cptr = p.chunk_ptr;

    // warp 0 stages chunk c into buffer b
    auto issue = [&](int64_t tile, int b) {
        const int64_t c = cbeg + tile;
        const int2 meta = sp.meta[c];
        const int64_t s0 = cptr[c];
        const unsigned nslot = static_cast<unsigned>(cptr[c + 1] - s0);
        unsigned char* base = smem_raw + b * stage_bytes;
        if (u == 0) {
            const unsigned total = static_cast<unsigned>(meta.y) * US * sizeof(T) +
                                   nslot * static_cast<unsigned>(sizeof(M)) + 1024 + 64;
            mbar_arrive_expect_tx(&bars[b], total);
            if (nslot) tma_load_1d(base + u_bytes, gvals + s0, nslot * sizeof(M), &bars[b]);
            tma_load_1d(base + u_bytes + v_bytes, sp.lcol + c * 512, 1024, &bars[b]);
            tma_load_1d(base + u_bytes + v_bytes + 1024, sp.lown + c * 32, 64, &bars[b]);
        }
        __syncwarp();
        for (int k = u; k < meta.x; k += 32) {
            const int4 run = sp.runs[c * kStageRuns + k];
            tma_load_1d(base + static_cast<size_t>(run.z) * US * sizeof(T),
                        in + static_cast<int64_t>(run.x) * pitch,
                        static_cast<unsigned>(run.y) * US * sizeof(T), &bars[b]);
        }
    };

    T wn[NP], xn[NP], x0n[NP];
    int64_t s0n = 0, s1n = 0;
    int fulln = 0;
    auto prefetch_rows = [&](int64_t tile) {
        const int64_t c = cbeg + tile;
        s0n = __ldg(&cptr[c]);
        s1n = __ldg(&cptr[c + 1]);
        fulln = __ldg(&p.chunk_full[c]);
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            const int64_t r = c * 32 + rr + i * R;
            if (r >= row0 && r < row1) {
                if constexpr (HAS_W) wn[i] = ld_stream(&W[r * pitch]);
                if constexpr (HAS_X) xn[i] = ld_stream(&X[r * pitch]);
                if constexpr (HAS_X0) x0n[i] = ld_stream(&X0[r * pitch]);
            }
        }
    };

    if (t == 0) {
        for (int b = 0; b < ns; ++b) mbar_init(&bars[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    int64_t tile = blockIdx.x;
    // prologue: stage the first ns - 1 tiles
    for (int b = 0; b + 1 < ns; ++b)
        if (rr == 0 && tile + b * static_cast<int64_t>(gridDim.x) < ntiles)
            issue(tile + b * static_cast<int64_t>(gridDim.x), b);
    if (tile < ntiles) prefetch_rows(tile);
    unsigned phases = 0u;
    for (int k = 0; tile < ntiles; ++k, tile += gridDim.x) {
        const int buf = k % ns;
        const bool more = tile + gridDim.x < ntiles;
        // refill the stage tile k - 1 used (every thread passed the barrier ending k - 1)
        const int64_t ahead = tile + static_cast<int64_t>(ns - 1) * gridDim.x;
        if (rr == 0 && ahead < ntiles) issue(ahead, (k + ns - 1) % ns);
        T wc[NP], xc[NP], x0c[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            wc[i] = wn[i];
            xc[i] = xn[i];
            x0c[i] = x0n[i];
        }
        const int64_t c = cbeg + tile;
        const int64_t s0 = s0n;
        const int w = static_cast<int>((s1n - s0) >> 5);
        const bool fast = w == MAXW && fulln != 0 && c * 32 >= row0 && c * 32 + 32 <= row1;
        if (more) prefetch_rows(tile + gridDim.x);
        mbar_wait(&bars[buf], (phases >> buf) & 1u);
        phases ^= 1u << buf;
        const T* us = U_s(buf);
        const M* vs = V_s(buf);
        const unsigned short* lcs = LC_s(buf);
        const unsigned short* los = LO_s(buf);
        // the warp's NP rows advance together: NP independent accumulation chains
        unsigned qw[NP][8];
        bool act[NP];
        T acc[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            const int l = rr + i * R;
            const int64_t r = c * 32 + l;
            act[i] = fast || (r >= row0 && r < row1);
            const uint4 q0 = *reinterpret_cast<const uint4*>(lcs + l * 16);  // broadcast
            const uint4 q1 = *reinterpret_cast<const uint4*>(lcs + l * 16 + 8);
            qw[i][0] = q0.x; qw[i][1] = q0.y; qw[i][2] = q0.z; qw[i][3] = q0.w;
            qw[i][4] = q1.x; qw[i][5] = q1.y; qw[i][6] = q1.z; qw[i][7] = q1.w;
            acc[i] = O::zero();
        }
        if (fast) {
#pragma unroll
            for (int j = 0; j < MAXW; ++j)
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    const unsigned lc = (qw[i][j >> 1] >> ((j & 1) * 16)) & 0xFFFFu;
                    acc[i] = O::vadd(acc[i], O::prod(vs[j * 32 + rr + i * R], us[lc * US + u]));
                }
        } else {
#pragma unroll
            for (int j = 0; j < MAXW; ++j)
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    const unsigned lc = (qw[i][j >> 1] >> ((j & 1) * 16)) & 0xFFFFu;
                    if (act[i] && j < w && lc != 0xFFFFu)
                        acc[i] = O::vadd(acc[i], O::prod(vs[j * 32 + rr + i * R], us[lc * US + u]));
                }
        }
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            if (!act[i]) continue;
            const int l = rr + i * R;
            const T ui = us[static_cast<int>(los[l]) * US + u];
            step_epilogue<O, T, KIND, DMODE>(acc[i], ui, wc[i], xc[i], x0c[i], (c * 32 + l) * pitch,
                                             W, X, X0, p.beta, coeff, c1, c2, acc_d, comp_d);
        }
        __syncthreads();  // stage `buf` is refilled by the next iteration's issue
    }

    if constexpr (NDOT > 0) {
        T acc_out[NDOT];
#pragma unroll
        for (int d = 0; d < NDOT; ++d) acc_out[d] = acc_d[d];
        void* outp = p.dots_out;
        const int64_t dstride = p.dots_row_stride;
        grid_reduce<T, NDOT>(acc_out, R, US, static_cast<T*>(p.partials), p.part_base + blockIdx.x,
                             p.nparts, p.final_launch != 0, p.counter,
                             [&](int d, int uu, T vv) {
                                 if (DMODE == 1)
                                     O::store_full(static_cast<T*>(outp), uu, vv);
                                 else
                                     O::store_re(static_cast<double*>(outp) + d * dstride, uu, vv);
                             });
    }
}

#endif  // CFD_EXPERIMENTAL

// ---- launch geometry -----------------------------------------------------------------------
struct Geometry {
    int US;      // units per row in this slab
    int R;       // rows per CTA iteration
    int threads;
};

inline Geometry geometry(int units) {
    Geometry g;
    g.US = units;
    g.R = units >= 256 ? 1 : 256 / units;
    g.threads = g.R * g.US;
    return g;
}

const void* find_scaled(const Matrix& a, double s) {
    for (const auto& e : a.scaled)
        if (e.first == s) return e.second->p;
    return nullptr;
}

// rows per CTA iteration as a power of two (tiles of whole 32-row chunks)
// CTA shape of the TMA kernel, measured on B200 (C1, C2, C3, graphene sweeps):
// on large operators small CTAs win -- the per-tile barrier waits on fewer
// warps -- 128 threads and 64-row tiles for rows of 8+ units, 64 threads for
// narrower rows; operators with fewer than 4 x SMs 64-row tiles (C1) keep
// 256-thread CTAs and 32-row tiles, or too few CTAs would run.
struct TmaShape {
    int cap_threads, tr, slab_max;
};
inline TmaShape tma_shape(const Context& ctx, int units, int64_t nrows) {
    if (nrows / 64 < 4 * static_cast<int64_t>(ctx.num_sms)) return {256, 32, 256};
    if (units <= 4) return {64, 64, 256};
    // rows wider than one CTA: 128-unit column slabs (C3 lattice, n_b = 256, with the
    // L2 hints: 128 / 64 / 32 / 16-unit slabs 19.8-20.9 / 19.9-20.2 / 20.1 / 20.9 ms
    // over two runs -- within run-to-run noise; wider slabs re-read the matrix less)
    return {128, 64, 128};
}
inline Geometry geometry_pow2(int units, int cap = CFD_TMA_THREADS) {
    Geometry g;
    g.US = units;
    int r = 1;
    while (r * 2 * units <= cap) r *= 2;
    g.R = r;
    g.threads = r * units;
    return g;
}

// Launch a step kernel, as a programmatic dependent of the previous kernel on the stream
// when `pdl` (the kernel calls griddepcontrol.wait before touching block vectors).
template <class K>
void launch_step_kernel(K kernel, int grid, int threads, size_t smem, cudaStream_t st, bool pdl,
                        const StepParams& p) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(static_cast<unsigned>(threads));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CFD_CUDA(cudaLaunchKernelEx(&cfg, kernel, p));
}

// Band (2.5D) tile order for lattice operators (Matrix::plane_rows > 0): the launch's
// rows are split into bands of whole lattice lines, each band swept plane by plane, so a
// tile's z -+ 1 neighbour rows were gathered one band slice earlier (a few MB) instead of
// one plane earlier (0.27-1 GB for C3/C4, beyond the L2).  The band is the largest
// divisor of the plane's lines whose slice of the gathered operand stays within
// ctx.band_bytes; operators whose whole plane fits keep row order.
inline uint64_t reciprocal64(uint64_t d) {  // ceil(2^64 / d), d >= 2
    return ~uint64_t(0) / d + 1;  // floor((2^64 - 1) / d) + 1 = ceil(2^64 / d) unless d | 2^64
}

inline void set_band_order(const Context& ctx, const Matrix& a, StepParams& p, int TR,
                           size_t row_bytes) {
    p.band_tps = 0;
    const int64_t P = a.plane_rows, Ln = a.line_rows;
    if (ctx.band_bytes <= 0 || P <= 0 || Ln <= 0 || P % Ln != 0) return;
    const int64_t rows = p.row1 - p.row0;
    if (rows <= 0 || p.row0 % P != 0 || rows % P != 0 || P % 32 != 0) return;
    // planes up to 4 slices (64 MB at the default) keep their z -+ 1 reuse in row order
    // (measured: C3 lattice n_b = 32, 32 MB planes, no gain; C4 share 1 GB and C3 n_b = 256
    // 128 MB slab planes -4 %, tools/band_exp.py)
    if (static_cast<size_t>(P) * row_bytes <= 4 * static_cast<size_t>(ctx.band_bytes)) return;
    if (rows / TR >= (int64_t(1) << 31)) return;  // 32-bit tile arithmetic
    const int64_t lines = P / Ln;
    int64_t by = 0;
    for (int64_t d = 1; d < lines; ++d)
        if (lines % d == 0 && (d * Ln) % TR == 0 &&
            static_cast<size_t>(d * Ln) * row_bytes <= static_cast<size_t>(ctx.band_bytes))
            by = d;
    if (by == 0) return;
    const int64_t slice = by * Ln;
    const uint64_t tps = static_cast<uint64_t>(slice / TR);
    const uint64_t per_band = static_cast<uint64_t>(rows / P) * tps;
    p.band_tps = static_cast<unsigned>(tps);
    p.band_per_band = static_cast<unsigned>(per_band);
    // ceil(2^64 / d) for d a power of two is 2^64 / d exactly, which the formula gives too
    // (d >= 2); d == 1 divides by identity in the kernel
    p.band_m_tps = tps >= 2 ? reciprocal64(tps) : 0;
    p.band_m_per_band = per_band >= 2 ? reciprocal64(per_band) : 0;
    p.band_plane_chunks = P / 32;
    p.band_slice_chunks = slice / 32;
}

template <class K>
int max_blocks_for(K kernel, int threads, size_t smem, int num_sms) {
    int per_sm = 0;
    CFD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
    return std::max(1, per_sm) * num_sms;
}

template <bool CPLX, class T, int KIND, int DMODE, int MAXW>
void run_step(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch) {
    const Matrix& a = *s.a;
    constexpr int NDOT = dots_of(DMODE);
    const int64_t nrows = s.row1 - s.row0;
    constexpr int MW = MAXW > 0 ? MAXW : 4;
    const void* svals = s.alpha == 1.0 ? a.vals.p : find_scaled(a, s.alpha);
    const bool tma = MAXW > 0 && ctx.kernel_variant >= 1 && svals != nullptr;
    auto kernel = tma ? step_tma_kernel<CPLX, T, KIND, DMODE, MW>
                      : step_kernel<CPLX, T, KIND, DMODE, 0>;
    int used_total = 0;
#if CFD_EXPERIMENTAL
    if constexpr (MAXW >= 8 && std::is_same_v<T, double2> && DMODE < 4) {
        // staged-gather kernel: one 512-byte row slot, plan present and fitting shared memory
        if (ctx.kernel_variant == 2 && tma && units == 32 && pitch == 32 && a.stage_max_rows > 0 &&
            nrows > 0) {
            const size_t stage = static_cast<size_t>(a.stage_max_rows) * 32 * sizeof(T) +
                                 32 * MAXW * sizeof(typename Ops<CPLX, T>::M) + 1024 + 64;
            const int nstage = 3 * stage <= 225 * 1024 ? 3 : 2;
            const size_t smem = nstage * stage;
            if (smem <= 225 * 1024) {
                auto sk = step_stage_kernel<CPLX, T, KIND, DMODE, MAXW>;
                static thread_local std::map<const void*, size_t> attr_set;
                auto& cur = attr_set[reinterpret_cast<const void*>(sk)];
                if (cur < smem) {
                    CFD_CUDA(cudaFuncSetAttribute(sk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  static_cast<int>(smem)));
                    cur = smem;
                }
                const int64_t need = ((s.row1 + 31) >> 5) - (s.row0 >> 5);
                const int grid =
                    static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, ctx.num_sms)));
                StepParams p{};
                p.chunk_ptr = a.chunk_ptr.as<int64_t>();
                p.chunk_full = a.chunk_full.as<unsigned char>();
                p.cols = a.cols.as<int>();
                p.vals = a.vals.p;
                p.svals = svals;
                p.row0 = s.row0;
                p.row1 = s.row1;
                p.halo_lo = a.part.halo_lo;
                p.pitch = pitch;
                p.u_off = 0;
                p.US = 32;
                p.R = 8;
                p.in = s.in;
                p.w = s.w;
                p.x = s.x;
                p.x0 = s.x0;
                p.alpha = s.alpha;
                p.beta = s.beta;
                p.c0 = s.c0;
                p.c1 = s.c1;
                p.c2 = s.c2;
                p.coeff_dev = s.coeff_dev;
                p.coeff_index = s.coeff_index;
                p.dots_out = s.dots_out;
                p.dots_row_stride = static_cast<int64_t>(units) * Ops<CPLX, T>::kCols;
                if (NDOT > 0) {
                    const size_t need_bytes =
                        static_cast<size_t>(reduce_rows_needed(s.partial_base + grid)) * NDOT * 32 * sizeof(T);
                    ctx.partials.ensure(std::max<size_t>(need_bytes, 1 << 20));
                    ctx.counter.ensure(4096);
                }
                p.partials = ctx.partials.p;
                p.part_base = s.partial_base;
                p.nparts = s.partial_base + grid;
                p.final_launch = s.final_launch ? 1 : 0;
                p.counter = ctx.counter.as<unsigned>();
                const StagePlan sp{a.stage_runs.as<int4>(), a.stage_meta.as<int2>(),
                                   a.stage_lcol.as<unsigned short>(),
                                   a.stage_lown.as<unsigned short>(), a.stage_max_rows, nstage};
                sk<<<grid, 256, smem, st>>>(p, sp);
                CFD_CUDA(cudaGetLastError());
                ctx.launches++;
                if (s.grid_used) *s.grid_used = grid;
                return;
            }
        }
    }
#endif  // CFD_EXPERIMENTAL
    if constexpr (MAXW > 0 && MAXW <= 8 && std::is_same_v<T, double2>) {
        // two units per thread: whole rows of 16 or 32 units (one chunk per tile)
        // default for short rows (graphene: +1..3 %, measured); TI's 11-entry rows keep
        // step_tma_kernel (the 2-unit gathers cost registers: 0.70 vs 0.61 ms on C2)
        const bool pick = ctx.kernel_variant == 3 || (ctx.kernel_variant == 1 && MAXW <= 8);
        if (pick && tma && units == pitch && (units == 16 || units == 32) && nrows > 0) {
            constexpr int NDOT2 = NDOT;
            constexpr bool HAS_W = kind_reads_w(KIND);
            constexpr bool HAS_X = kind_reads_x(KIND);
            constexpr bool HAS_X0 = (DMODE == 2 && KIND != kStepStart2);
            constexpr int NS = (HAS_W ? 1 : 0) + (HAS_X ? 1 : 0) + (HAS_X0 ? 1 : 0);
            using M = typename Ops<CPLX, T>::M;
            const size_t cap = static_cast<size_t>(MAXW) * 32;
            const size_t stage = ((cap * sizeof(int) + 15) & ~size_t(15)) + cap * sizeof(M) +
                                 static_cast<size_t>(NS) * 32 * pitch * sizeof(T);
            const int HS = units / 2, R = 256 / HS;
            const size_t smem = std::max(2 * stage, static_cast<size_t>(NDOT2) * 256 * 2 * sizeof(T));
            auto k2 = step_tma2_kernel<CPLX, KIND, DMODE, MAXW>;
            if (smem > 48 * 1024) {
                static thread_local std::map<const void*, size_t> attr_set;
                auto& cur = attr_set[reinterpret_cast<const void*>(k2)];
                if (cur < smem) {
                    CFD_CUDA(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  static_cast<int>(smem)));
                    cur = smem;
                }
            }
            static thread_local std::map<std::pair<const void*, size_t>, int> occ2;
            auto key = std::make_pair(reinterpret_cast<const void*>(k2), smem);
            auto it = occ2.find(key);
            const int maxb = it != occ2.end() ? it->second
                                              : (occ2[key] = max_blocks_for(k2, 256, smem, ctx.num_sms));
            const int64_t need = ((s.row1 + 31) >> 5) - (s.row0 >> 5);
            const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, maxb)));
            StepParams p{};
            p.chunk_ptr = a.chunk_ptr.as<int64_t>();
            p.chunk_full = a.chunk_full.as<unsigned char>();
            p.cols = a.cols.as<int>();
            p.vals = a.vals.p;
            p.svals = svals;
            p.row0 = s.row0;
            p.row1 = s.row1;
            p.halo_lo = a.part.halo_lo;
            p.pitch = pitch;
            p.u_off = 0;
            p.US = units;
            p.R = R;
            p.in = s.in;
            p.w = s.w;
            p.x = s.x;
            p.x0 = s.x0;
            p.alpha = s.alpha;
            p.beta = s.beta;
            p.c0 = s.c0;
            p.c1 = s.c1;
            p.c2 = s.c2;
            p.coeff_dev = s.coeff_dev;
            p.coeff_index = s.coeff_index;
            p.dots_out = s.dots_out;
            p.dots_row_stride = static_cast<int64_t>(units) * Ops<CPLX, T>::kCols;
            if (NDOT > 0) {
                const size_t need_bytes =
                    static_cast<size_t>(reduce_rows_needed(s.partial_base + grid)) * NDOT * units * sizeof(T);
                ctx.partials.ensure(std::max<size_t>(need_bytes, 1 << 20));
                ctx.counter.ensure(4096);
            }
            p.partials = ctx.partials.p;
            p.part_base = s.partial_base;
            p.nparts = s.partial_base + grid;
            p.final_launch = s.final_launch ? 1 : 0;
            p.counter = ctx.counter.as<unsigned>();
            launch_step_kernel(k2, grid, 256, smem, st,
                               s.pdl_ok && (ctx.pdl == 2 || (ctx.pdl == 1 && nrows / 64 < 4 * static_cast<int64_t>(ctx.num_sms))),
                               p);
            CFD_CUDA(cudaGetLastError());
            ctx.launches++;
            if (s.grid_used) *s.grid_used = grid;
            return;
        }
    }
    // column slabs of at most `slab` units (one CTA row-group spans a slab)
    const TmaShape shape = tma_shape(ctx, units, nrows);
    const int slab_max = tma ? shape.slab_max : 256;  // one CTA row-group spans a slab
    const int slab = ctx.slab_units > 0 ? std::min(ctx.slab_units, slab_max) : slab_max;
    for (int u0 = 0; u0 < units; u0 += slab) {
        const int us = std::min(slab, units - u0);
        Geometry g = tma ? geometry_pow2(us, shape.cap_threads) : geometry(us);
        const int TR = std::max(tma ? shape.tr : 32, g.R);
        const size_t stage = tma ? 2 * static_cast<size_t>(MW) * TR : 0;
        size_t ring = tma ? ((stage * sizeof(int) + 15) & ~size_t(15)) + stage * (CPLX ? 16 : 8)
                          : 0;
        // the TMA kernel's shared dot accumulators follow the ring (modes 2-4)
        if (tma && NDOT > 0 && DMODE != 1)
            ring = ((ring + 15) & ~size_t(15)) + NDOT * static_cast<size_t>(g.threads) * sizeof(T);
        const size_t smem = std::max(NDOT * static_cast<size_t>(g.threads) * sizeof(T), ring);
        if (smem > 48 * 1024) {
            static thread_local std::map<const void*, size_t> attr_set;
            auto& cur = attr_set[reinterpret_cast<const void*>(kernel)];
            if (cur < smem) {
                CFD_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              static_cast<int>(smem)));
                cur = smem;
            }
        }
        static thread_local std::map<std::tuple<const void*, int, size_t>, int> occ_cache;
        auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), g.threads, smem);
        auto it = occ_cache.find(key);
        int maxb = 0;
        if (it == occ_cache.end()) {
            maxb = max_blocks_for(kernel, g.threads, smem, ctx.num_sms);
            occ_cache[key] = maxb;
        } else {
            maxb = it->second;
        }
        const int64_t need = tma ? (((s.row1 + 31) >> 5) - (s.row0 >> 5) + TR / 32 - 1) / (TR / 32)
                                 : (nrows + g.R - 1) / g.R;
        int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, maxb)));
        StepParams p{};
        p.chunk_ptr = a.chunk_ptr.as<int64_t>();
        p.chunk_full = a.chunk_full.as<unsigned char>();
        p.cols = a.cols.as<int>();
        p.vals = a.vals.p;
        p.svals = svals;
        p.row0 = s.row0;
        p.row1 = s.row1;
        p.halo_lo = a.part.halo_lo;
        p.pitch = pitch;
        p.u_off = u0;
        p.US = us;
        p.R = g.R;
        p.in = s.in;
        p.w = s.w;
        p.x = s.x;
        p.x0 = s.x0;
        p.alpha = s.alpha;
        p.beta = s.beta;
        p.c0 = s.c0;
        p.c1 = s.c1;
        p.c2 = s.c2;
        p.coeff_dev = s.coeff_dev;
        p.coeff_index = s.coeff_index;
        p.dots_out = s.dots_out;
        p.dots_row_stride = static_cast<int64_t>(units) * Ops<CPLX, T>::kCols;  // = nb columns
        if (NDOT > 0) {
            const size_t need_bytes =
                static_cast<size_t>(reduce_rows_needed(s.partial_base + grid)) * NDOT * us * sizeof(T);
            // partials are slab-local: slabs run sequentially on the stream
            ctx.partials.ensure(std::max<size_t>(need_bytes, 1 << 20));
            ctx.counter.ensure(4096);
        }
        p.partials = ctx.partials.p;
        p.part_base = s.partial_base;
        p.nparts = s.partial_base + grid;
        p.final_launch = s.final_launch ? 1 : 0;
        p.counter = ctx.counter.as<unsigned>();
        p.tr = TR;
        p.band_tps = 0;
        p.tile_a = 1;
        auto launch_kernel = kernel;
        // band (2.5D) order for dot-free steps on lattice operators with planes beyond the
        // L2 budget: a non-persistent grid of ctx.tiles_per_cta tiles per CTA (ORDER 1)
        if constexpr (CPLX && DMODE == 0 && MAXW == 11) {
            if (tma && ctx.tiles_per_cta > 0) {
                set_band_order(ctx, a, p, TR, static_cast<size_t>(us) * sizeof(T));
                if (p.band_tps != 0) {
                    const int64_t tpc = ctx.tiles_per_cta;
                    grid = static_cast<int>((need + tpc - 1) / tpc);
                    p.tile_a = tpc;
                    launch_kernel = step_tma_kernel<CPLX, T, KIND, DMODE, MW, 1>;
                    if (nrows > 0) ++ctx.band_launches;
                    if (smem > 48 * 1024)
                        CFD_CUDA(cudaFuncSetAttribute(launch_kernel,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      static_cast<int>(smem)));
                }
            }
        }
        if (nrows > 0) {
            // PDL pays where launches dominate (C1: 4.2 -> 3.6 us per step); on operators of
            // 4 x SMs tiles or more it measured neutral to -2 % (C2, C5), so only there
            const bool pdl = tma && s.pdl_ok &&
                             (ctx.pdl == 2 || (ctx.pdl == 1 && nrows / 64 < 4 * static_cast<int64_t>(ctx.num_sms)));
            launch_step_kernel(launch_kernel, grid, g.threads, smem, st, pdl, p);
            CFD_CUDA(cudaGetLastError());
            ctx.launches++;
        }
        used_total = grid;
        if (units > slab && NDOT > 0 && !s.final_launch)
            fail(CHEBFD_ERR_UNSUPPORTED, "split dot launches need a single column slab");
    }
    if (s.grid_used) *s.grid_used = used_total;
}

template <bool CPLX, class T, int MAXW>
void dispatch_kind_w(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch) {
    switch (s.kind_step) {
        case kStepSpmmvm:
            if (s.dots_mode == 3) return run_step<CPLX, T, kStepSpmmvm, 3, MAXW>(ctx, s, st, units, pitch);
            if (s.dots_mode == 4) return run_step<CPLX, T, kStepSpmmvm, 4, MAXW>(ctx, s, st, units, pitch);
            return run_step<CPLX, T, kStepSpmmvm, 0, MAXW>(ctx, s, st, units, pitch);
        case kStepStart2:
            if (s.dots_mode == 2) return run_step<CPLX, T, kStepStart2, 2, MAXW>(ctx, s, st, units, pitch);
            if (s.dots_mode == 4) return run_step<CPLX, T, kStepStart2, 4, MAXW>(ctx, s, st, units, pitch);
            return run_step<CPLX, T, kStepStart2, 0, MAXW>(ctx, s, st, units, pitch);
        case kStepFused:
            if (s.dots_mode == 1) return run_step<CPLX, T, kStepFused, 1, MAXW>(ctx, s, st, units, pitch);
            if (s.dots_mode == 2) return run_step<CPLX, T, kStepFused, 2, MAXW>(ctx, s, st, units, pitch);
            if (s.dots_mode == 4) return run_step<CPLX, T, kStepFused, 4, MAXW>(ctx, s, st, units, pitch);
            return run_step<CPLX, T, kStepFused, 0, MAXW>(ctx, s, st, units, pitch);
        case kStepFusedX2:
            if (s.dots_mode == 2) return run_step<CPLX, T, kStepFusedX2, 2, MAXW>(ctx, s, st, units, pitch);
            if (s.dots_mode == 0) return run_step<CPLX, T, kStepFusedX2, 0, MAXW>(ctx, s, st, units, pitch);
            break;
        case kStepFusedX3:
            if (s.dots_mode == 2) return run_step<CPLX, T, kStepFusedX3, 2, MAXW>(ctx, s, st, units, pitch);
            if (s.dots_mode == 0) return run_step<CPLX, T, kStepFusedX3, 0, MAXW>(ctx, s, st, units, pitch);
            break;
        case kStepRecur:
            if (s.dots_mode == 2) return run_step<CPLX, T, kStepRecur, 2, MAXW>(ctx, s, st, units, pitch);
            if (s.dots_mode == 4) return run_step<CPLX, T, kStepRecur, 4, MAXW>(ctx, s, st, units, pitch);
            if (s.dots_mode == 5) return run_step<CPLX, T, kStepRecur, 5, MAXW>(ctx, s, st, units, pitch);
            if (s.dots_mode == 6) return run_step<CPLX, T, kStepRecur, 6, MAXW>(ctx, s, st, units, pitch);
            return run_step<CPLX, T, kStepRecur, 0, MAXW>(ctx, s, st, units, pitch);
    }
    fail(CHEBFD_ERR_INVALID_ARGUMENT, "bad step kind");
}

// Row-width buckets: graphene rows have 4 entries, TI rows 10-11.
template <bool CPLX, class T>
void dispatch_kind(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch) {
    const int w = s.a->max_row_len;
    if (w <= 4) return dispatch_kind_w<CPLX, T, 4>(ctx, s, st, units, pitch);
    if (w <= 8) return dispatch_kind_w<CPLX, T, 8>(ctx, s, st, units, pitch);
    if (w <= 11) return dispatch_kind_w<CPLX, T, 11>(ctx, s, st, units, pitch);
    if (w <= 16) return dispatch_kind_w<CPLX, T, 16>(ctx, s, st, units, pitch);
    return dispatch_kind_w<CPLX, T, 0>(ctx, s, st, units, pitch);
}

}  // namespace
}  // namespace cfd
