// Two Chebyshev steps per launch: a wavefront over the row space that keeps
// the intermediate vector in L2 ("pair kernel").
//
// apply_filter's fused loop (filter.hpp:105-114, kernels.hpp:74-118) streams
// five block vectors per step: U gathered, W read + written, X read + written.
// Two consecutive steps n, n+1 are
//     W <- 2(aA+b)U - W      (= V_n,     phase 1)
//     U <- 2(aA+b)W - U      (= V_{n+1}, phase 2)
//     X <- (X + c_n V_n) + c_{n+1} V_{n+1}
// Row r of phase 2 needs V_n only on rows within the operator's bandwidth b
// of r.  One persistent launch therefore walks the rows in order: work item i
// runs phase 1 on row tile i and phase 2 on tile i - L, where L exceeds the
// bandwidth (in tiles) plus the tiles in flight.  V_n is written by phase 1
// and gathered by phase 2 a few planes later -- from L2 -- and X is read and
// written once per pair.  Per pair the block streams drop from 10 to 6 (plus
// the matrix once instead of twice).
//
// Ordering, all on the device:
//  * items are claimed in increasing order from a ticket counter, so every
//    tile phase 2 waits on was claimed earlier by a running CTA, whose phase 1
//    never waits: no deadlock whatever the residency;
//  * phase 1 of a tile publishes its chunk count into a per-group counter
//    (release); phase 2 of tile j waits (acquire) until every group covering
//    rows [j*TR - b, (j+1)*TR + b) is complete.  That also orders phase 2's
//    in-place overwrite of U after every phase-1 gather of those rows;
//  * the last CTA to leave resets the counters (graph replays need no memset).
//
// Every element is computed with the reference's operations in the
// reference's order (the same Ops as the single-step kernels), so W, U and X
// stay bit-identical to two spmmvm_fused calls.  The moments of both steps,
// <x0, V_n> and <x0, V_{n+1}>, are reduced in phase 2 (one x0 read).
#include <cuda_runtime.h>

#include <algorithm>
#include <map>

#ifndef CFD_TMA_THREADS
#define CFD_TMA_THREADS 256
#endif
#ifndef CFD_TMA_MINB
#define CFD_TMA_MINB 2
#endif

#include "internal.hpp"
#include "step_common.cuh"

namespace cfd {

#if CFD_EXPERIMENTAL  // opt-in variant, measured slower; not in the default build

namespace {

constexpr int kGroupChunksLog2 = 5;  // 32 chunks (1024 rows) per completion group

struct PairParams {
    StepParams p;     // in = U (V_{n-1}), w = W (V_{n-2}); alpha, beta already doubled
    unsigned* sync;   // [0] item ticket, [1] exit ticket, [2 + g] chunks of group g done
    int ntiles;       // row tiles of TR rows
    int lag;          // L: phase 2 trails phase 1 by this many tiles
    int64_t band;     // max |column - row| of the operator (rows)
    int nchunks;
    int hints;        // L2 eviction-priority hints on (1) / off (0)
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// coherent, L1-cached loads: V_n and U are written during this launch, so the
// read-only (.nc) path of the single-step kernels is not allowed here
__device__ __forceinline__ double ld_coh(const double* p) { return __ldca(p); }
__device__ __forceinline__ double2 ld_coh(const double2* p) { return __ldca(p); }

// L2 eviction priorities: the wavefront keeps V_n (and the matrix rows of the
// window) in L2 while the read-once / write-once streams pass through
__device__ __forceinline__ uint64_t l2_policy(bool keep, bool hints) {
    uint64_t pol;
    if (!hints)
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    else if (keep)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double ld_hint(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double2 ld_hint(const double2* p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(double2* p, double2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y),
                 "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, unsigned bytes,
                                                 uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

template <bool CPLX, class T, int DMODE, int MAXW>
__global__ void __launch_bounds__(CFD_TMA_THREADS, CFD_TMA_MINB) step_pair_kernel(const PairParams q) {
    using O = Ops<CPLX, T>;
    using M = typename O::M;
    constexpr int NDOT = DMODE == 2 ? 2 : 0;
    const StepParams& p = q.p;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[2];
    __shared__ int s_item[2];
    __shared__ unsigned s_last;
    const int t = threadIdx.x;
    const int US = p.US;
    const int rr = t / US;
    const int u = t - rr * US;
    const int R = p.R;
    const int TR = R > p.tr ? R : p.tr;
    const int NCH = TR / 32;
    const int cap = MAXW * TR;  // slots per tile buffer; 4 buffers: (item buffer) x (phase)
    int* cols_s = reinterpret_cast<int*>(smem_raw);
    M* vals_s = reinterpret_cast<M*>(smem_raw + ((4 * cap * sizeof(int) + 15) & ~size_t(15)));

    const int cu = p.u_off + u;
    T* __restrict__ U = static_cast<T*>(const_cast<void*>(p.in)) + cu;  // extended base
    T* __restrict__ W = static_cast<T*>(p.w) + cu;
    T* __restrict__ X = static_cast<T*>(p.x) + cu;
    const T* __restrict__ X0 = static_cast<const T*>(p.x0) + cu;
    const M* __restrict__ gvals = static_cast<const M*>(p.svals);
    const int pitch = p.pitch;
    const int64_t halo = p.halo_lo;
    const double c1 = p.coeff_dev[p.coeff_index];
    const double c2 = p.coeff_dev[p.coeff_index + 1];
    const double beta = p.beta;
    const int64_t nrows = p.row1;  // row0 == 0: single-rank operators only
    const int ntiles = q.ntiles, L = q.lag;
    const int nitems = ntiles + L;
    const int nch = q.nchunks;
    const int64_t* __restrict__ cptr = p.chunk_ptr;
    unsigned* const ticket = q.sync;
    unsigned* const done = q.sync + 2;

    T acc_d[NDOT > 0 ? NDOT : 1];
#pragma unroll
    for (int d = 0; d < (NDOT > 0 ? NDOT : 1); ++d) acc_d[d] = O::zero();
    const uint64_t pol_keep = l2_policy(true, q.hints != 0);
    const uint64_t pol_stream = l2_policy(false, q.hints != 0);

    auto issue = [&](int item, int buf) {
        unsigned bytes = 0;
        int64_t rng[2][2];
        int tiles[2] = {item < ntiles ? item : -1, (item - L >= 0 && item - L < ntiles) ? item - L : -1};
        for (int ph = 0; ph < 2; ++ph) {
            rng[ph][0] = rng[ph][1] = 0;
            if (tiles[ph] < 0) continue;
            const int64_t c0 = static_cast<int64_t>(tiles[ph]) * NCH;
            const int64_t c1e = min(c0 + NCH, static_cast<int64_t>(nch));
            rng[ph][0] = cptr[c0];
            rng[ph][1] = cptr[c1e];
            bytes += static_cast<unsigned>(rng[ph][1] - rng[ph][0]) * (4u + sizeof(M));
        }
        mbar_arrive_expect_tx(&bars[buf], bytes);
        for (int ph = 0; ph < 2; ++ph) {
            const unsigned n = static_cast<unsigned>(rng[ph][1] - rng[ph][0]);
            if (!n) continue;
            const int slot = (2 * buf + ph) * cap;
            const uint64_t pol = ph == 0 ? pol_keep : pol_stream;  // phase 2 reads it last
            tma_load_1d_hint(cols_s + slot, p.cols + rng[ph][0], n * 4u, &bars[buf], pol);
            tma_load_1d_hint(vals_s + slot, gvals + rng[ph][0], n * static_cast<unsigned>(sizeof(M)),
                             &bars[buf], pol);
        }
    };

    // one row of phase PH (1: W <- f(U) - W;  2: U <- f(W) - U, X, moments)
    auto row = [&](auto ph_tag, auto fast_tag, int64_t r, int64_t c0, int64_t sbase, const int* cs,
                   const M* vs) {
        constexpr int PH = decltype(ph_tag)::value;
        constexpr bool FAST = decltype(fast_tag)::value;
        const T* __restrict__ in = PH == 1 ? U : W;  // gathered operand (extended rows)
        T* __restrict__ out = PH == 1 ? W : U;       // updated in place (owned rows)
        const int lane = static_cast<int>(r & 31);
        int coff, w;
        if constexpr (FAST) {
            coff = static_cast<int>((r >> 5) - c0) * (32 * MAXW) + lane;
            w = MAXW;
        } else {
            const int64_t chunk = r >> 5;
            const int64_t cb = __ldg(&cptr[chunk]);
            coff = static_cast<int>(cb - sbase) + lane;
            w = static_cast<int>((__ldg(&cptr[chunk + 1]) - cb) >> 5);
        }
        const int64_t own = r * pitch;
        const T wi = ld_hint(&out[own], pol_stream);  // V_{n-2} / V_{n-1}: last use
        T xi{}, x0v{};
        if constexpr (PH == 2) {
            xi = ld_hint(&X[own], pol_stream);
            if constexpr (DMODE == 2) x0v = ld_hint(&X0[own], pol_stream);
        }
        T acc = O::zero();
        int c[MAXW];
#pragma unroll
        for (int j = 0; j < MAXW; ++j) c[j] = (FAST || j < w) ? cs[coff + j * 32] : -1;
        T g[MAXW];
#pragma unroll
        for (int j = 0; j < MAXW; ++j)
            if (FAST || c[j] >= 0) g[j] = ld_coh(&in[static_cast<int64_t>(c[j]) * pitch]);
#pragma unroll
        for (int j = 0; j < MAXW; ++j)
            if (FAST || c[j] >= 0) acc = O::vadd(acc, O::prod(vs[coff + j * 32], g[j]));
        const T ui = ld_coh(&in[(r + halo) * pitch]);
        const T wn = O::vsub(O::vadd(acc, O::smul(beta, ui)), wi);  // kernels.hpp:103
        if constexpr (PH == 1) {
            st_hint(&out[own], wn, pol_keep);  // V_n: gathered by phase 2 a few planes later
        } else {
            st_hint(&out[own], wn, pol_stream);
            // X += c_n V_n; X += c_{n+1} V_{n+1}  (kernels.hpp:106, twice, same roundings)
            st_hint(&X[own], O::vadd(O::vadd(xi, O::smul(c1, ui)), O::smul(c2, wn)), pol_stream);
            if constexpr (DMODE == 2) {
                acc_d[0] = O::vadd(acc_d[0], O::cdot(x0v, ui));
                acc_d[1] = O::vadd(acc_d[1], O::cdot(x0v, wn));
            }
        }
    };

    auto tile_rows = [&](auto ph_tag, int tile, const int* cs, const M* vs) {
        const int64_t c0 = static_cast<int64_t>(tile) * NCH;
        const int64_t c1e = min(c0 + NCH, static_cast<int64_t>(nch));
        const int64_t sbase = cptr[c0];
        bool fast = (cptr[c1e] - sbase) == (c1e - c0) * 32 * MAXW && c1e * 32 <= nrows &&
                    (c1e - c0) == NCH;
        for (int64_t c = c0; fast && c < c1e; ++c) fast = __ldg(&p.chunk_full[c]) != 0;
        if (fast) {
            for (int it = 0; it < TR; it += R)
                row(ph_tag, std::true_type{}, c0 * 32 + it + rr, c0, sbase, cs, vs);
        } else {
            for (int it = 0; it < TR; it += R) {
                const int64_t r = c0 * 32 + it + rr;
                if (r >= nrows) continue;
                row(ph_tag, std::false_type{}, r, c0, sbase, cs, vs);
            }
        }
    };

    if (t == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        const int first = static_cast<int>(atomicAdd(ticket, 1u));
        s_item[0] = first;
        if (first < nitems) issue(first, 0);
    }
    __syncthreads();
    int item = s_item[0];
    unsigned phases = 0u;
    for (int k = 0; item < nitems; ++k) {
        const int buf = k & 1;
        if (t == 0) {
            const int next = static_cast<int>(atomicAdd(ticket, 1u));
            s_item[buf ^ 1] = next;
            if (next < nitems) issue(next, buf ^ 1);
        }
        mbar_wait(&bars[buf], (phases >> buf) & 1u);
        phases ^= 1u << buf;
        // phase 1 on tile `item`
        if (item < ntiles) {
            tile_rows(std::integral_constant<int, 1>{}, item, cols_s + (2 * buf) * cap,
                      vals_s + (2 * buf) * cap);
            __syncthreads();
            if (t == 0) {
                const int64_t c0 = static_cast<int64_t>(item) * NCH;
                const unsigned n = static_cast<unsigned>(min(c0 + NCH, static_cast<int64_t>(nch)) - c0);
                __threadfence();
                atomicAdd(&done[c0 >> kGroupChunksLog2], n);
            }
        }
        // phase 2 on tile item - L, once phase 1 covered its rows +- band
        const int j = item - L;
        if (j >= 0 && j < ntiles) {
            const int64_t r_lo = max(static_cast<int64_t>(j) * TR - q.band, int64_t{0});
            const int64_t r_hi = min((static_cast<int64_t>(j) + 1) * TR + q.band, nrows) - 1;
            const int g_lo = static_cast<int>((r_lo >> 5) >> kGroupChunksLog2);
            const int g_hi = static_cast<int>((r_hi >> 5) >> kGroupChunksLog2);
            for (int g = g_lo + t; g <= g_hi; g += blockDim.x) {
                const unsigned want =
                    static_cast<unsigned>(min(nch - (g << kGroupChunksLog2), 1 << kGroupChunksLog2));
                while (ld_acquire(&done[g]) < want) __nanosleep(64);
            }
            __threadfence();
            __syncthreads();
            tile_rows(std::integral_constant<int, 2>{}, j, cols_s + (2 * buf + 1) * cap,
                      vals_s + (2 * buf + 1) * cap);
        }
        __syncthreads();  // buffer `buf` is refilled next iteration; s_item visible
        item = s_item[buf ^ 1];
    }

    if constexpr (NDOT > 0) {
        T acc_out[NDOT];
#pragma unroll
        for (int d = 0; d < NDOT; ++d) acc_out[d] = acc_d[d];
        const int uoff = p.u_off;
        void* outp = p.dots_out;
        const int64_t dstride = p.dots_row_stride;
        grid_reduce<T, NDOT>(acc_out, R, US, static_cast<T*>(p.partials), blockIdx.x, gridDim.x, true,
                             p.counter, [&](int d, int uu, T vv) {
                                 O::store_re(static_cast<double*>(outp) + d * dstride, uoff + uu, vv);
                             });
    }
    // the last CTA out resets the tickets and group counters for the next launch
    __syncthreads();
    if (t == 0) {
        __threadfence();
        s_last = atomicAdd(&q.sync[1], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        const int ngroups = (nch + (1 << kGroupChunksLog2) - 1) >> kGroupChunksLog2;
        for (int g = t; g < ngroups; g += blockDim.x) done[g] = 0u;
        if (t == 0) {
            q.sync[0] = 0u;
            q.sync[1] = 0u;
        }
    }
}

const void* scaled_copy(const Matrix& a, double s) {
    for (const auto& e : a.scaled)
        if (e.first == s) return e.second->p;
    return nullptr;
}

template <bool CPLX, class T, int DMODE, int MAXW>
bool run_pair(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch) {
    const Matrix& a = *s.a;
    constexpr int NDOT = DMODE == 2 ? 2 : 0;
    using M = typename Ops<CPLX, T>::M;
    const int64_t nrows = s.row1 - s.row0;
    const void* svals = scaled_copy(a, s.alpha);
    if (!svals || nrows <= 0 || s.row0 != 0 || a.part.halo_lo != 0 || a.part.halo_hi != 0)
        return false;
    const int nch = static_cast<int>((nrows + 31) >> 5);
    const size_t groups = (static_cast<size_t>(nch) + 31) >> kGroupChunksLog2;
    if (a.pair_sync.bytes < sizeof(unsigned) * (2 + groups)) return false;
    const bool small = nrows / 64 < 4 * static_cast<int64_t>(ctx.num_sms);
    auto kernel = step_pair_kernel<CPLX, T, DMODE, MAXW>;

    // launch geometry for column slabs of w units
    struct Plan {
        int R, threads, TR, grid, ntiles, lag;
        size_t smem;
        double ws;  // bytes the wavefront touches between the phases of a row
    };
    auto plan = [&](int w, Plan& g) -> bool {
        const int cap_threads = ctx.pair_threads > 0 ? ctx.pair_threads : (small ? 256 : 128);
        if (w > cap_threads) return false;
        g.R = 1;
        while (g.R * 2 * w <= cap_threads) g.R *= 2;
        g.threads = g.R * w;
        g.TR = std::max(ctx.pair_tile_rows > 0 ? ctx.pair_tile_rows : (small ? 32 : 64), g.R);
        const size_t cap = static_cast<size_t>(MAXW) * g.TR;
        const size_t ring = ((4 * cap * sizeof(int) + 15) & ~size_t(15)) + 4 * cap * sizeof(M);
        g.smem = std::max(ring, static_cast<size_t>(NDOT) * g.threads * sizeof(T));
        static thread_local std::map<const void*, size_t> attr_set;
        auto& cur = attr_set[reinterpret_cast<const void*>(kernel)];
        if (g.smem > 40 * 1024 && cur < g.smem) {  // + static shared memory: opt in early
            CFD_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(g.smem)));
            cur = g.smem;
        }
        static thread_local std::map<std::tuple<const void*, int, size_t>, int> occ;
        auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), g.threads, g.smem);
        auto it = occ.find(key);
        int per_sm = 0;
        if (it == occ.end()) {
            CFD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, g.threads, g.smem));
            occ[key] = per_sm;
        } else {
            per_sm = it->second;
        }
        if (per_sm < 1) return false;
        g.ntiles = (nch + g.TR / 32 - 1) / (g.TR / 32);
        g.grid = static_cast<int>(std::min<int64_t>(g.ntiles, static_cast<int64_t>(per_sm) * ctx.num_sms));
        // phase 2 trails by the bandwidth (in tiles) plus the tiles in flight; it waits on
        // whole 1024-row groups, so every tile it can wait on must have been claimed before
        // (lag > band + one group), or all CTAs could end up waiting
        const int64_t band_tiles = (a.band + g.TR - 1) / g.TR + 1;
        const int extra = ctx.pair_extra >= 0 ? ctx.pair_extra : g.grid;
        const int64_t min_lag = band_tiles + (32 / (g.TR / 32)) + 1;
        g.lag = static_cast<int>(std::min<int64_t>(min_lag + extra, g.ntiles));
        // between a row's phase 1 and its last phase-2 reader the wavefront advances
        // lag tiles + band rows; per row it touches U, W (twice), X (twice) and the matrix
        const double rows_between =
            std::min<double>(static_cast<double>(g.lag) * g.TR + a.band, static_cast<double>(nrows));
        const double mat_row =
            static_cast<double>(a.entries) / std::max<int64_t>(nrows, 1) * (4.0 + sizeof(M));
        g.ws = rows_between * (5.0 * w * sizeof(T) + mat_row);
        return true;
    };

    if (ctx.pair_mode == 1) {
        // measured on B200: on operators whose blocks stream from HBM the
        // step kernel is latency-bound, not byte-bound, and the pair kernel loses (C2:
        // 0.83 vs 0.62 ms per step); it pays where the whole filter state is L2-resident
        // and launches dominate
        const double foot = static_cast<double>(nrows) * units * sizeof(T) * (NDOT > 0 ? 4 : 3) +
                            static_cast<double>(a.entries) * (4.0 + sizeof(M));
        if (foot > 0.5 * ctx.l2_bytes) return false;
    }
    // slab width: forced, else the widest whose wavefront fits the L2 (narrower slabs
    // re-read the matrix once per slab)
    int w = 0;
    Plan g{};
    if (ctx.pair_slab > 0) {
        w = std::min(ctx.pair_slab, units);
        if (!plan(w, g)) return false;
    } else {
        for (int cand = units; cand >= 1; cand = (cand + 1) / 2) {
            Plan c{};
            if (plan(cand, c) && (ctx.pair_mode == 2 || c.ws <= 0.6 * ctx.l2_bytes)) {
                w = cand;
                g = c;
                break;
            }
            if (cand == 1 || cand < 4) break;
        }
        if (w == 0) return false;
    }
    if (NDOT > 0) {
        ctx.partials.ensure(
            std::max<size_t>(static_cast<size_t>(reduce_rows_needed(g.grid)) * NDOT * units * sizeof(T),
                             1 << 20));
        ctx.counter.ensure(4096);
    }
    for (int u0 = 0; u0 < units; u0 += w) {
        PairParams q{};
        StepParams& p = q.p;
        p.chunk_ptr = a.chunk_ptr.as<int64_t>();
        p.chunk_full = a.chunk_full.as<unsigned char>();
        p.cols = a.cols.as<int>();
        p.vals = a.vals.p;
        p.svals = svals;
        p.row0 = 0;
        p.row1 = nrows;
        p.halo_lo = a.part.halo_lo;
        p.pitch = pitch;
        p.u_off = u0;
        p.US = std::min(w, units - u0);
        Plan gs = g;
        if (p.US != w && !plan(p.US, gs)) fail(CHEBFD_ERR_CUDA, "pair kernel: no geometry for the last slab");
        p.R = gs.R;
        p.in = s.in;
        p.w = s.w;
        p.x = s.x;
        p.x0 = s.x0;
        p.alpha = s.alpha;
        p.beta = s.beta;
        p.coeff_dev = s.coeff_dev;
        p.coeff_index = s.coeff_index;
        p.dots_out = s.dots_out;
        p.dots_row_stride = static_cast<int64_t>(units) * Ops<CPLX, T>::kCols;
        p.partials = ctx.partials.p;
        p.counter = ctx.counter.as<unsigned>();
        p.tr = gs.TR;
        q.sync = a.pair_sync.as<unsigned>();
        q.ntiles = gs.ntiles;
        q.lag = gs.lag;
        q.band = a.band;
        q.nchunks = nch;
        q.hints = ctx.pair_hints;
        kernel<<<gs.grid, gs.threads, gs.smem, st>>>(q);
        CFD_CUDA(cudaGetLastError());
        ctx.launches++;
        if (s.grid_used) *s.grid_used = gs.grid;
    }
    return true;
}

template <bool CPLX, class T, int MAXW>
bool pair_dmode(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch) {
    if (s.dots_mode == 2) return run_pair<CPLX, T, 2, MAXW>(ctx, s, st, units, pitch);
    if (s.dots_mode == 0) return run_pair<CPLX, T, 0, MAXW>(ctx, s, st, units, pitch);
    return false;
}

template <bool CPLX, class T>
bool pair_width(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch) {
    const int w = s.a->max_row_len;
    if (w <= 4) return pair_dmode<CPLX, T, 4>(ctx, s, st, units, pitch);
    if (w <= 8) return pair_dmode<CPLX, T, 8>(ctx, s, st, units, pitch);
    if (w <= 11) return pair_dmode<CPLX, T, 11>(ctx, s, st, units, pitch);
    if (w <= 16) return pair_dmode<CPLX, T, 16>(ctx, s, st, units, pitch);
    return false;
}

}  // namespace

bool launch_step_pair(Context& ctx, const StepArgs& s, cudaStream_t st) {
    const int kind = s.a->kind;
    const int64_t width = s.width_cols;
    if (kind == CHEBFD_COMPLEX128)
        return pair_width<true, double2>(ctx, s, st, static_cast<int>(width), static_cast<int>(width));
    if (width % 2 == 0)
        return pair_width<false, double2>(ctx, s, st, static_cast<int>(width / 2),
                                          static_cast<int>(width / 2));
    return pair_width<false, double>(ctx, s, st, static_cast<int>(width), static_cast<int>(width));
}

#else
bool launch_step_pair(Context&, const StepArgs&, cudaStream_t) { return false; }
#endif  // CFD_EXPERIMENTAL

}  // namespace cfd
