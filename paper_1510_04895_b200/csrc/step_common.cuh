// Device building blocks shared by the step kernels (kernels.cu, pair.cu):
// the reference-order fp64 arithmetic (Ops), fixed-order grid reductions,
// the step parameter block, and the TMA / mbarrier helpers.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "internal.hpp"

namespace cfd {
namespace {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double div_(double a, double b) { return __ddiv_rn(a, b); }

template <class T>
__device__ __forceinline__ T ldg(const T* p) { return __ldg(p); }

// Streaming loads/stores (evict-first) for the read-once / write-once streams.
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(double* p, double v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double2* p, double2 v) { __stcs(p, v); }

// ---- scalar traits: (complex?, unit type) ------------------------------------------
template <bool CPLX, class T>
struct Ops;

// real, one column per unit
template <>
struct Ops<false, double> {
    using M = double;
    static constexpr int kCols = 1;
    __device__ static double zero() { return 0.0; }
    __device__ static M scale(M a, double s) { return mul(a, s); }
    __device__ static double prod(M a, double u) { return mul(a, u); }
    __device__ static double vadd(double a, double b) { return add(a, b); }
    __device__ static double vsub(double a, double b) { return sub(a, b); }
    __device__ static double smul(double s, double v) { return mul(s, v); }
    __device__ static double cdot(double x, double w) { return mul(x, w); }
    using DT = double;  // moment / plain-dot accumulator
    __device__ static double cdot_re(double x, double w) { return mul(x, w); }
    __device__ static double lam_mul(const double* lam, int col, double v) { return mul(lam[col], v); }
    __device__ static double cdiv(double v, const double* d, int col) { return div_(v, d[col]); }
    __device__ static void store_re(double* out, int unit, double v) { out[unit] = v; }
    __device__ static void store_full(double* out, int unit, double v) { out[unit] = v; }
};

// real, two columns per unit
template <>
struct Ops<false, double2> {
    using M = double;
    static constexpr int kCols = 2;
    __device__ static double2 zero() { return make_double2(0.0, 0.0); }
    __device__ static M scale(M a, double s) { return mul(a, s); }
    __device__ static double2 prod(M a, double2 u) { return make_double2(mul(a, u.x), mul(a, u.y)); }
    __device__ static double2 vadd(double2 a, double2 b) { return make_double2(add(a.x, b.x), add(a.y, b.y)); }
    __device__ static double2 vsub(double2 a, double2 b) { return make_double2(sub(a.x, b.x), sub(a.y, b.y)); }
    __device__ static double2 smul(double s, double2 v) { return make_double2(mul(s, v.x), mul(s, v.y)); }
    __device__ static double2 cdot(double2 x, double2 w) { return make_double2(mul(x.x, w.x), mul(x.y, w.y)); }
    using DT = double2;  // two real columns: both products are moments
    __device__ static double2 cdot_re(double2 x, double2 w) { return cdot(x, w); }
    __device__ static double2 lam_mul(const double* lam, int col, double2 v) {
        return make_double2(mul(lam[col], v.x), mul(lam[col + 1], v.y));
    }
    __device__ static double2 cdiv(double2 v, const double* d, int col) {
        return make_double2(div_(v.x, d[col]), div_(v.y, d[col + 1]));
    }
    __device__ static void store_re(double* out, int unit, double2 v) {
        out[2 * unit] = v.x;
        out[2 * unit + 1] = v.y;
    }
    __device__ static void store_full(double2* out, int unit, double2 v) { out[unit] = v; }
};

// complex, one column per unit (std::complex<double> layout)
template <>
struct Ops<true, double2> {
    using M = double2;
    static constexpr int kCols = 1;
    __device__ static double2 zero() { return make_double2(0.0, 0.0); }
    // complex * double (libstdc++ operator*(complex, T): componentwise)
    __device__ static M scale(M a, double s) { return make_double2(mul(a.x, s), mul(a.y, s)); }
    // complex * complex, GCC inline expansion: (ac - bd, ad + bc)
    __device__ static double2 prod(M a, double2 u) {
        return make_double2(sub(mul(a.x, u.x), mul(a.y, u.y)), add(mul(a.x, u.y), mul(a.y, u.x)));
    }
    __device__ static double2 vadd(double2 a, double2 b) { return make_double2(add(a.x, b.x), add(a.y, b.y)); }
    __device__ static double2 vsub(double2 a, double2 b) { return make_double2(sub(a.x, b.x), sub(a.y, b.y)); }
    __device__ static double2 smul(double s, double2 v) { return make_double2(mul(s, v.x), mul(s, v.y)); }
    // conj(x) * w
    __device__ static double2 cdot(double2 x, double2 w) {
        const double nxi = -x.y;
        return make_double2(sub(mul(x.x, w.x), mul(nxi, w.y)), add(mul(x.x, w.y), mul(nxi, w.x)));
    }
    // Re(conj(x) w) alone (moments are real parts): the same bits as cdot(x, w).x
    using DT = double;
    __device__ static double cdot_re(double2 x, double2 w) {
        const double nxi = -x.y;
        return sub(mul(x.x, w.x), mul(nxi, w.y));
    }
    __device__ static void store_re(double* out, int unit, double v) { out[unit] = v; }
    __device__ static double2 lam_mul(const double* lam, int col, double2 v) { return smul(lam[col], v); }
    __device__ static double2 cdiv(double2 v, const double* d, int col) {
        return make_double2(div_(v.x, d[col]), div_(v.y, d[col]));
    }
    __device__ static void store_re(double* out, int unit, double2 v) { out[unit] = v.x; }
    __device__ static void store_full(double2* out, int unit, double2 v) { out[unit] = v; }
};

template <class T>
__device__ __forceinline__ void kahan_add(T& s, T& c, T v);
template <>
__device__ __forceinline__ void kahan_add<double>(double& s, double& c, double v) {
    const double y = sub(v, c);
    const double t = add(s, y);
    c = sub(sub(t, s), y);
    s = t;
}
template <>
__device__ __forceinline__ void kahan_add<double2>(double2& s, double2& c, double2 v) {
    kahan_add<double>(s.x, c.x, v.x);
    kahan_add<double>(s.y, c.y, v.y);
}

template <class T>
__device__ __forceinline__ T tadd(T a, T b);
template <>
__device__ __forceinline__ double tadd<double>(double a, double b) { return add(a, b); }
template <>
__device__ __forceinline__ double2 tadd<double2>(double2 a, double2 b) {
    return make_double2(add(a.x, b.x), add(a.y, b.y));
}

// L2-coherent load of a partial (double, double2, or a pair of double2 units)
template <class T>
__device__ __forceinline__ T ldcg_t(const T* p) {
    if constexpr (std::is_same_v<T, double> || std::is_same_v<T, double2>) {
        return __ldcg(p);
    } else {
        const double2* q = reinterpret_cast<const double2*>(p);
        return T{__ldcg(q), __ldcg(q + 1)};
    }
}

// dot products a step accumulates: 1 Kahan <x,w> / 2 <x0,w> / 3 m0,m1 + x0 copy /
// 4 moment pair / 5 moment quad / 6 the quad's upper pair (doubling identities)
__host__ __device__ constexpr int dots_of(int dmode) {
    return dmode == 0 ? 0 : (dmode == 5 ? 4 : (dmode >= 3 ? 2 : 1));
}

// ---- step kinds: which own-row streams a kind reads ----------------------------------
__host__ __device__ constexpr bool kind_reads_w(int k) {
    return k == kStepFused || k == kStepRecur || k == kStepFusedX2 || k == kStepFusedX3;
}
__host__ __device__ constexpr bool kind_reads_x(int k) {
    return k == kStepFused || k == kStepStart2 || k == kStepFusedX2 || k == kStepFusedX3;
}
__host__ __device__ constexpr bool kind_fused(int k) {
    return k == kStepFused || k == kStepFusedX2 || k == kStepFusedX3;
}

// ---- fixed-order block + grid reduction of NDOT per-unit accumulators -------------
// Threads are laid out t = rr*US + u.  Each CTA writes NDOT*US partials.  When all
// partials come from this launch, the last CTA of every group of kReduceGroup CTAs sums
// its group's partials in index order, and the last group to finish sums the group
// sums in order (two short reductions instead of one CTA reading every partial while
// the GPU idles).  A launch that completes partials of earlier launches
// (interior + boundary rows) sums rows [0, nparts) in order in its last CTA.  Either
// way the order -- hence every bit -- is fixed, and `emit(d, u, value)` gets the totals.
// counter[0]: grid ticket, counter[1 + g]: group tickets; all self-resetting.
constexpr int kReduceGroup = 32;
// partial rows a grid reduction over n CTA partials needs (its group sums included)
__host__ __device__ constexpr int64_t reduce_rows_needed(int64_t n) { return n + (n + kReduceGroup - 1) / kReduceGroup; }

// GUARD: the CTA has more than R * US threads (the site-ring kernel's producer warps); the
// extra threads only take part in the barriers.
template <class T, int NDOT, bool GUARD = false, class Emit>
__device__ __forceinline__ void grid_reduce(const T (&acc)[NDOT > 0 ? NDOT : 1], int R, int US,
                                            T* partials, int part_slot, int nparts, bool final_launch,
                                            unsigned* counter, Emit emit) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sred = reinterpret_cast<T*>(smem_raw);
    const int t = threadIdx.x;
    const int rr = t / US, u = t - rr * US;
    const int nthr = R * US;
    const bool part = !GUARD || t < nthr;
    if (part) {
#pragma unroll
        for (int d = 0; d < NDOT; ++d) sred[d * nthr + t] = acc[d];
    }
    __syncthreads();
    if (rr == 0) {
#pragma unroll
        for (int d = 0; d < NDOT; ++d) {
            T s = sred[d * nthr + u];
            for (int q = 1; q < R; ++q) s = tadd(s, sred[d * nthr + q * US + u]);
            partials[(static_cast<int64_t>(part_slot) * NDOT + d) * US + u] = s;
        }
    }
    if (!final_launch) return;
    __threadfence();
    __syncthreads();
    __shared__ unsigned is_last;
    // rows [first, first + count) of src (NDOT x US each) summed in index order; the
    // totals land in sred[d * nthr + u] (rr == 0 threads hold them after the call)
    auto reduce_rows = [&](const T* src, int first, int count) {
#pragma unroll
        for (int d = 0; d < NDOT; ++d) {
            // rows rr, rr + R, rr + 2R, ... left to right, eight loads in flight
            auto at = [&](int q) {
                return ldcg_t(&src[(static_cast<int64_t>(first + q) * NDOT + d) * US + u]);
            };
            if (!part) continue;
            T s = T{};
            int q = rr;
            if (q < count) {
                s = at(q);
                q += R;
            }
            for (; q + 7 * R < count; q += 8 * R) {
                T v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) v[k] = at(q + k * R);
#pragma unroll
                for (int k = 0; k < 8; ++k) s = tadd(s, v[k]);
            }
            for (; q < count; q += R) s = tadd(s, at(q));
            sred[d * nthr + t] = s;
        }
        __syncthreads();
        if (rr == 0) {
#pragma unroll
            for (int d = 0; d < NDOT; ++d) {
                T s = sred[d * nthr + u];
                const int lim = R < count ? R : count;
                for (int q = 1; q < lim; ++q) s = tadd(s, sred[d * nthr + q * US + u]);
                sred[d * nthr + u] = s;
            }
        }
    };
    const bool two_level = nparts == static_cast<int>(gridDim.x) && part_slot == static_cast<int>(blockIdx.x);
    if (two_level) {
        const int g = static_cast<int>(blockIdx.x) / kReduceGroup;
        const int gsize = min(kReduceGroup, nparts - g * kReduceGroup);
        const int ngroups = (nparts + kReduceGroup - 1) / kReduceGroup;
        if (t == 0) is_last = (atomicAdd(&counter[1 + g], 1u) == static_cast<unsigned>(gsize - 1));
        __syncthreads();
        if (!is_last) return;
        __threadfence();
        T* gpart = partials + static_cast<int64_t>(nparts) * NDOT * US;
        reduce_rows(partials, g * kReduceGroup, gsize);
        if (rr == 0) {
#pragma unroll
            for (int d = 0; d < NDOT; ++d)
                gpart[(static_cast<int64_t>(g) * NDOT + d) * US + u] = sred[d * nthr + u];
        }
        __threadfence();
        __syncthreads();
        if (t == 0) {
            counter[1 + g] = 0u;
            is_last = (atomicAdd(counter, 1u) == static_cast<unsigned>(ngroups - 1));
        }
        __syncthreads();
        if (!is_last) return;
        __threadfence();
        reduce_rows(gpart, 0, ngroups);
    } else {
        if (t == 0) is_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
        __syncthreads();
        if (!is_last) return;
        __threadfence();
        reduce_rows(partials, 0, nparts);
    }
    if (rr == 0) {
#pragma unroll
        for (int d = 0; d < NDOT; ++d) emit(d, u, sred[d * nthr + u]);
    }
    if (t == 0) *counter = 0u;  // self-reset for the next stream-ordered launch
}

// ---- the Chebyshev step kernel --------------------------------------------------------
struct StepParams {
    const int64_t* chunk_ptr;
    const unsigned char* chunk_full;  // 1: every row of the chunk has exactly `width` entries
    const int* cols;
    const void* vals;
    const void* svals;    // values pre-multiplied by `alpha` (or null)
    int64_t row0, row1;   // owned rows of this launch
    int64_t halo_lo;      // extended-row offset of owned row 0
    int pitch;            // units per row in memory
    int u_off;            // first unit of this column slab
    int US;               // units in this slab (threads per row)
    int R;                // rows per CTA iteration
    const void* in;       // gathered operand (extended base)
    void* w;              // owned base
    void* x;
    void* x0;
    double alpha, beta;   // already 2x for start2/fused/recur
    double c0, c1, c2;
    const double* coeff_dev;
    int coeff_index;
    void* dots_out;
    int64_t dots_row_stride;  // doubles between the NDOT output rows (moment rows)
    void* partials;
    int part_base;
    int nparts;
    int final_launch;
    unsigned* counter;
    int tr;  // minimum rows per tile of the TMA kernels (32 or 64)
    // band (2.5D) tile order of the TMA kernel for lattice operators: the
    // launch's rows are whole lattice planes of band_plane_chunks chunks; tiles enumerate
    // (band, plane, tile in the band's slice of the plane), so the z -+ 1 planes a tile
    // gathers were touched one slice (not one plane) earlier.  band_tps = 0: row order.
    // Divisions by the invariant tiles-per-band / tiles-per-slice use host-computed
    // reciprocals M = ceil(2^64 / d) (exact for 32-bit numerators), so the mapping costs
    // a few multiplies and no registers in the row loop.
    unsigned band_tps;          // tiles per band slice (0: row order)
    unsigned band_per_band;     // tiles per band (planes x band_tps)
    uint64_t band_m_tps, band_m_per_band;
    int64_t band_plane_chunks;  // 32-row chunks per plane
    int64_t band_slice_chunks;  // 32-row chunks per band slice
    int64_t tile_a;             // tiles per CTA of a non-persistent (ORDER 1) launch
};

// n / d for 32-bit n with the host reciprocal m = ceil(2^64 / d) (d >= 2), or n (d == 1)
__device__ __forceinline__ unsigned div_by(unsigned n, unsigned d, uint64_t m) {
    return d == 1u ? n : static_cast<unsigned>(__umul64hi(static_cast<uint64_t>(n), m));
}

// first chunk of tile `tile` of a launch starting at chunk cbeg (NCH chunks per tile)
__device__ __forceinline__ int64_t tile_first_chunk(const StepParams& p, int64_t tile, int64_t cbeg,
                                                    int NCH) {
    if (p.band_tps == 0u) return cbeg + tile * NCH;
    const unsigned tl = static_cast<unsigned>(tile);
    const unsigned b = div_by(tl, p.band_per_band, p.band_m_per_band);
    const unsigned rem = tl - b * p.band_per_band;
    const unsigned z = div_by(rem, p.band_tps, p.band_m_tps);
    const unsigned j = rem - z * p.band_tps;
    return cbeg + static_cast<int64_t>(z) * p.band_plane_chunks +
           static_cast<int64_t>(b) * p.band_slice_chunks + static_cast<int64_t>(j) * NCH;
}

// Sum_j (a_rj * scale) * in[c_rj] over one row, in the row's stored order.
// MAXW > 0: all column indices of the row are loaded first, then every
// gather is issued before the first use (maximum memory-level parallelism).
template <class O, class T, class M, int MAXW>
__device__ __forceinline__ T gather_row(const int* __restrict__ cols, const M* __restrict__ vals,
                                        const T* __restrict__ in, int64_t base, int width, int lane,
                                        int pitch, int64_t col_off, double scale) {
    T acc = O::zero();
    if constexpr (MAXW > 0) {
        int c[MAXW];
#pragma unroll
        for (int j = 0; j < MAXW; ++j)
            c[j] = (j < width) ? __ldg(&cols[base + static_cast<int64_t>(j) * 32 + lane]) : -1;
        T g[MAXW];
#pragma unroll
        for (int j = 0; j < MAXW; ++j)
            if (c[j] >= 0) g[j] = ldg(&in[static_cast<int64_t>(c[j]) * pitch + col_off]);
#pragma unroll
        for (int j = 0; j < MAXW; ++j)
            if (c[j] >= 0) {
                const M v = __ldg(&vals[base + static_cast<int64_t>(j) * 32 + lane]);
                acc = O::vadd(acc, O::prod(O::scale(v, scale), g[j]));
            }
    } else {
        constexpr int BATCH = 8;
        for (int j0 = 0; j0 < width; j0 += BATCH) {
            int c[BATCH];
            T g[BATCH];
#pragma unroll
            for (int b = 0; b < BATCH; ++b)
                c[b] = (j0 + b < width) ? __ldg(&cols[base + static_cast<int64_t>(j0 + b) * 32 + lane]) : -1;
#pragma unroll
            for (int b = 0; b < BATCH; ++b)
                if (c[b] >= 0) g[b] = ldg(&in[static_cast<int64_t>(c[b]) * pitch + col_off]);
#pragma unroll
            for (int b = 0; b < BATCH; ++b)
                if (c[b] >= 0) {
                    const M v = __ldg(&vals[base + static_cast<int64_t>(j0 + b) * 32 + lane]);
                    acc = O::vadd(acc, O::prod(O::scale(v, scale), g[b]));
                }
        }
    }
    return acc;
}

// Per-entry epilogue of each step kind, in the reference's operation order.
// Moment doubling (DMODE 4): for Hermitian h, V_n = T_n(h) x0 gives
//   <x0, T_{2n} x0> = 2 <V_n, V_n> - <x0, x0>,  <x0, T_{2n+1} x0> = 2 <V_n, V_{n+1}> - <x0, T_1 x0>
// so the step producing V_{n+1} from V_n (own row ui, result wn) yields the raw sums for
// moments 2n and 2n+1 from registers: no x0 stream, and only the first half of a filter's
// steps reduce at all.  The host applies 2 raw - m0 / 2 raw - m1 (capi.cu).
// acc += <x, w> in the accumulator's type: the full product for unit-typed (T)
// accumulators, its real part alone for O::DT ones (same bits as the product's .x)
template <class O, class A, class T>
__device__ __forceinline__ void dot_acc(A& acc, const T x, const T w) {
    if constexpr (std::is_same_v<A, T>)
        acc = O::vadd(acc, O::cdot(x, w));
    else
        acc = add(acc, O::cdot_re(x, w));
}

template <class O, class A, class T, int NA>
__device__ __forceinline__ void moment_pair(A (&acc_d)[NA], const T ui, const T wn) {
    dot_acc<O>(acc_d[0], ui, ui);
    dot_acc<O>(acc_d[1], ui, wn);
}

// Four moments from one recurrence step (DMODE 5): the step producing V_n holds V_{n-2}
// (wi), V_{n-1} (ui) and V_n (wn) in registers, whose products give the raw sums of
// moments 2n-3 (<V_{n-2},V_{n-1}>), 2n-2, 2n-1 and 2n (<V_n,V_n>).  With the delayed X
// update every second step is such a V_n-only step, so the X-update steps reduce nothing.
template <class O, class A, class T, int NA>
__device__ __forceinline__ void moment_quad(A (&acc_d)[NA], const T wi, const T ui, const T wn) {
    dot_acc<O>(acc_d[0], wi, ui);
    dot_acc<O>(acc_d[1], ui, ui);
    dot_acc<O>(acc_d[2], ui, wn);
    dot_acc<O>(acc_d[3], wn, wn);
}

template <class O, class T, int KIND, int DMODE, class A, int NA>
__device__ __forceinline__ void step_epilogue(const T acc, const T ui, const T wi, const T xi,
                                              const T x0v, int64_t own, T* __restrict__ W,
                                              T* __restrict__ X, T* __restrict__ X0, double beta,
                                              double coeff, double c1, double c2, A (&acc_d)[NA],
                                              A (&comp_d)[NA]) {
    if constexpr (KIND == kStepSpmmvm) {
        T y = acc;
        if (beta != 0.0) y = O::vadd(y, O::smul(beta, ui));  // kernels.hpp:62-65
        st_stream(&W[own], y);
        if constexpr (DMODE == 3 || DMODE == 4) {  // filter entry: m0 = <x,x>, m1 = <x,u>
            if constexpr (DMODE == 3) st_stream(&X0[own], ui);  // x0 = X (direct moments)
            dot_acc<O>(acc_d[0], ui, ui);
            dot_acc<O>(acc_d[1], ui, y);
        }
    } else if constexpr (KIND == kStepStart2) {
        // w = spmmvm(A,u,2a,2b); w = 1*w + (-1)*x + 0*x; x = c0 x + c1 u + c2 w  (filter.hpp:93-103)
        T wr = acc;
        if (beta != 0.0) wr = O::vadd(wr, O::smul(beta, ui));
        const T wn = O::vadd(O::vadd(O::smul(1.0, wr), O::smul(-1.0, xi)), O::smul(0.0, xi));
        st_stream(&W[own], wn);
        if constexpr (DMODE == 2) dot_acc<O>(acc_d[0], xi, wn);
        if constexpr (DMODE == 4) moment_pair<O>(acc_d, ui, wn);
        const T xn = O::vadd(O::vadd(O::smul(coeff, xi), O::smul(c1, ui)), O::smul(c2, wn));
        st_stream(&X[own], xn);
    } else {
        // fused / recur: w' = tmp + 2b u_i - w_i  (kernels.hpp:103,142)
        const T wn = O::vsub(O::vadd(acc, O::smul(beta, ui)), wi);
        st_stream(&W[own], wn);
        if constexpr (KIND == kStepFused) {
            if constexpr (DMODE == 1) kahan_add<T>(acc_d[0], comp_d[0], O::cdot(xi, wn));
            if constexpr (DMODE == 2) dot_acc<O>(acc_d[0], x0v, wn);
            st_stream(&X[own], O::vadd(xi, O::smul(coeff, wn)));  // kernels.hpp:106
        } else if constexpr (KIND == kStepFusedX2) {
            // the previous step's X += c_{n-1} V_{n-1} (ui) and this step's X += c_n V_n,
            // in that order: the reference's two roundings (kernels.hpp:106, twice)
            if constexpr (DMODE == 2) dot_acc<O>(acc_d[0], x0v, wn);
            st_stream(&X[own], O::vadd(O::vadd(xi, O::smul(c1, ui)), O::smul(coeff, wn)));
        } else if constexpr (KIND == kStepFusedX3) {
            // X += c_{n-2} V_{n-2} (wi), c_{n-1} V_{n-1} (ui), c_n V_n, in that order
            if constexpr (DMODE == 2) dot_acc<O>(acc_d[0], x0v, wn);
            st_stream(&X[own], O::vadd(O::vadd(O::vadd(xi, O::smul(c2, wi)), O::smul(c1, ui)),
                                       O::smul(coeff, wn)));
        } else {
            if constexpr (DMODE == 2) dot_acc<O>(acc_d[0], x0v, wn);
        }
        if constexpr (DMODE == 4) moment_pair<O>(acc_d, ui, wn);
        if constexpr (DMODE == 5) moment_quad<O>(acc_d, wi, ui, wn);
        if constexpr (DMODE == 6) {  // the upper pair of moment_quad: moments 2n-1, 2n
            dot_acc<O>(acc_d[0], ui, wn);
            dot_acc<O>(acc_d[1], wn, wn);
        }
    }
}

// ---- L2 eviction-priority hints (createpolicy + .L2::cache_hint) -------------------
// mode 0: evict_normal, 1: evict_last, 2: evict_first
__device__ __forceinline__ uint64_t l2_make_policy(int mode) {
    uint64_t pol;
    if (mode == 1)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else if (mode == 2)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// read-only (nc) load with an L2 policy
__device__ __forceinline__ double ldg_pol(const double* p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double2 ldg_pol(const double2* p, uint64_t pol) {
    double2 v;
    asm("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}
// coherent streaming load (no L1 allocation) with an L2 policy
__device__ __forceinline__ double lds_pol(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double2 lds_pol(const double2* p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}

// ---- TMA bulk copies and mbarriers -------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LAB_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra LAB_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

}  // namespace
}  // namespace cfd
