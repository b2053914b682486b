// Row-group step kernel (sm_100a): the default step kernel where the matrix has a grouped
// form (internal.hpp GroupedMatrix; built by group.cu).
//
// A thread owns one 16-byte unit of FOUR consecutive rows (a lattice site's orbitals): the
// group's merged column list is gathered once and every gathered unit feeds all the rows
// that reference it from registers.  On the TI operator a site's 44 entries touch 24
// distinct neighbour rows, so a step moves 24 + 4 (own rows) instead of 44 + 4 row units
// through the L1 per site, and reads 24 packed column words + 44 values from shared memory
// instead of 44 + 44 -- the SELL kernel's limit was L1 throughput, not HBM.
// Each row still meets its entries in CSR order: W and X are bit-identical to the SELL
// kernels and to the reference.
//
// Tiles are 16 groups (64 rows): header + packed columns and the values arrive in shared
// memory by two TMA bulk copies per tile, double-buffered (as step_tma_kernel).  The row
// mask of a column is warp-uniform whenever a row spans a whole warp (32+ units), so the
// four "does row r take this column" tests are uniform branches.
#pragma once
#include <utility>

#include "group_patterns.hpp"
#include "step_kernels.cuh"

#ifndef CFD_GRP_THREADS
#define CFD_GRP_THREADS 128
#endif
#ifndef CFD_GRP_X_EARLY
#define CFD_GRP_X_EARLY 1  // X rows loaded with W (16 registers) instead of after the products:
                           // C4 X-update step 9.50 -> 8.87 ms (alternating A/B)
#endif
#ifndef CFD_GRP_MINB
#define CFD_GRP_MINB 2  // 255 registers per thread (8 warps/SM): a site's 24 gathers, W and
                        // the hoisted matrix values in flight.  168 registers (12 warps/SM,
                        // ~50 bytes spilled) measured slower in an alternating A/B on one box:
                        // C4 filter 7.94 vs 7.78 ms per step, X-update steps 10.9 vs 9.5 ms
#endif

namespace cfd {
namespace {

template <class F, int... I>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, I...>) {
    (f(std::integral_constant<int, I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
    static_for_impl(f, std::make_integer_sequence<int, N>{});
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

struct GroupParams {
    const int64_t* tile_cptr;
    const int64_t* tile_vptr;
    const int* cols;
    const void* vals;  // pre-multiplied by alpha
    int cap_c;         // ints per shared-memory stage
    int cap_v;         // values per stage
    TileMap tm;        // tile -> rows (linear or line-interleaved)
};

// Measured dead ends on B200 (tools/group_exp.py): per-column row tests as
// branches, predicates or a 16-way jump (generic path: 0.58-1.1 ms per C2 step against
// 0.47 ms for the SELL kernel); software pipelining over groups with a second register
// buffer or at half-group granularity (spills at 255 registers); L1 / L2 prefetch of the
// next group's rows (+-3 %); tiles of 2 or 4 lattice lines (no gain).
template <bool CPLX, class T, int KIND, int DMODE, int ORDER>
__global__ void __launch_bounds__(CFD_GRP_THREADS, CFD_GRP_MINB)
    step_group_kernel(const StepParams p, const GroupParams gp) {
    using O = Ops<CPLX, T>;
    using M = typename O::M;
    constexpr int NDOT = dots_of(DMODE);
    constexpr int G = kGroupRows;
    constexpr int NCH = kTileRows / 32;
    constexpr int NH = 12;  // gathers per register half
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[2];
    const int t = threadIdx.x;
    const int US = p.US;
    const int rr = t / US;
    const int u = t - rr * US;
    const int R = p.R;  // groups per pass
    int* cols_s = reinterpret_cast<int*>(smem_raw);
    M* vals_s = reinterpret_cast<M*>(smem_raw + 2 * static_cast<size_t>(gp.cap_c) * sizeof(int));
    constexpr bool SACC = NDOT > 0 && DMODE != 1;
    using A = std::conditional_t<DMODE == 1, T, typename O::DT>;
    A* sacc = reinterpret_cast<A*>(smem_raw + 2 * static_cast<size_t>(gp.cap_c) * sizeof(int) +
                                   2 * static_cast<size_t>(gp.cap_v) * sizeof(M));

    const int cu = p.u_off + u;
    const T* __restrict__ inu = static_cast<const T*>(p.in) + cu;
    T* __restrict__ W = static_cast<T*>(p.w) + cu;
    T* __restrict__ X = static_cast<T*>(p.x) + cu;
    T* __restrict__ X0 = static_cast<T*>(p.x0) + cu;
    const M* __restrict__ gvals = static_cast<const M*>(gp.vals);
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
    A acc_d[NDOT > 0 ? NDOT : 1];
    A comp_d[NDOT > 0 ? NDOT : 1];
#pragma unroll
    for (int d = 0; d < (NDOT > 0 ? NDOT : 1); ++d) {
        acc_d[d] = A{};
        comp_d[d] = A{};
    }
    const uint64_t pol_keep = l2_make_policy(1);
    const uint64_t pol_stream = l2_make_policy(2);
    const int64_t row0 = p.row0, row1 = p.row1;
    const int64_t cbeg = row0 >> 5;  // row0 is a multiple of the tile (launcher)
    const int64_t cend = (row1 + 31) >> 5;
    const int64_t ntiles = row1 > row0 ? (cend - cbeg + NCH - 1) / NCH : 0;

    auto first_chunk = [&](int64_t tile) -> int64_t {
        if constexpr (ORDER == 0)
            return cbeg + tile * NCH;
        else
            return tile_first_chunk(p, tile, cbeg, NCH);
    };
    auto issue = [&](int64_t tile, int buf) {
        const int64_t tt = first_chunk(tile) / NCH;
        const int64_t a0 = gp.tile_cptr[tt], a1 = gp.tile_cptr[tt + 1];
        const int64_t v0 = gp.tile_vptr[tt], v1 = gp.tile_vptr[tt + 1];
        const unsigned bc = static_cast<unsigned>(a1 - a0) * 4u;
        const unsigned bv = static_cast<unsigned>(v1 - v0) * static_cast<unsigned>(sizeof(M));
        mbar_arrive_expect_tx(&bars[buf], bc + bv);
        tma_load_1d(cols_s + buf * gp.cap_c, gp.cols + a0, bc, &bars[buf]);
        if (bv) tma_load_1d(vals_s + buf * gp.cap_v, gvals + v0, bv, &bars[buf]);
    };
    auto ldgk = [&](const T* q) { return ldg_pol(q, pol_keep); };
    auto ldst = [&](const T* q) { return lds_pol(q, pol_stream); };
    auto col_of = [&](int c) {
        return static_cast<int64_t>(static_cast<unsigned>(c) & 0x0FFFFFFFu) * pitch;
    };

    // ---- pieces of one group (rows rg .. rg + 3, owned indices) --------------------------
    // Rows outside [row0, row1) (ragged launch edges) load from the nearest row inside and
    // skip their epilogue, so there is a single code path.
    struct Rows {
        bool ok[G];
        int64_t own[G];
    };
    auto rows_of = [&](int64_t rg) {
        Rows q;
#pragma unroll
        for (int r = 0; r < G; ++r) {
            q.ok[r] = rg + r >= row0 && rg + r < row1;
            q.own[r] = min(max(rg + r, row0), row1 - 1) * pitch;
        }
        return q;
    };
    // W and X now; x0 is read after the products and only starts towards the L2 here
    auto load_w = [&](const Rows& q, T (&wi)[G], T (&xi)[G]) {
#pragma unroll
        for (int r = 0; r < G; ++r) {
            wi[r] = xi[r] = T{};
            if constexpr (kind_reads_w(KIND)) wi[r] = ldst(&W[q.own[r]]);
            if constexpr (kind_reads_x(KIND)) {
                if constexpr (CFD_GRP_X_EARLY)
                    xi[r] = ldst(&X[q.own[r]]);
                else
                    prefetch_l2(&X[q.own[r]]);
            }
            if constexpr (DMODE == 2 && KIND != kStepStart2) prefetch_l2(&X0[q.own[r]]);
        }
    };
    // half `hf` (12 gathers) of static-pattern group gi of the staged tile `seg`
    auto gather_half = [&](T (&g)[NH], int gi, const int* seg, int hf) {
        const int4 h = reinterpret_cast<const int4*>(seg)[gi];
        const int4* cq = reinterpret_cast<const int4*>(seg + h.x) + hf * (NH / 4);
#pragma unroll
        for (int q = 0; q < NH / 4; ++q) {
            const int4 c4 = cq[q];
            g[4 * q] = ldgk(&inu[col_of(c4.x)]);
            g[4 * q + 1] = ldgk(&inu[col_of(c4.y)]);
            g[4 * q + 2] = ldgk(&inu[col_of(c4.z)]);
            g[4 * q + 3] = ldgk(&inu[col_of(c4.w)]);
        }
    };
    // products of half HF of pattern P: values at fixed offsets of the group's stream
    auto mac_half = [&](auto pat_tag, auto half_tag, const T (&g)[NH], const M* vs, T (&acc)[G],
                        T (&ui)[G]) {
        using P = decltype(pat_tag);
        constexpr int HF = decltype(half_tag)::value;
        static_for<NH>([&](auto kt) {
            constexpr int k = HF * NH + decltype(kt)::value;
            if constexpr (k < P::NC) {
                static_for<G>([&](auto rt) {
                    constexpr int r = decltype(rt)::value;
                    if constexpr ((P::m(k) >> r) & 1u) {
                        const M v = vs[P::voff(k, r)];
                        const T gk = g[k - HF * NH];
                        if constexpr (!CPLX) {
                            acc[r] = O::vadd(acc[r], O::prod(v, gk));
                        } else if constexpr ((P::re(k) >> r) & 1u) {
                            acc[r].x = add(acc[r].x, mul(v.x, gk.x));
                            acc[r].y = add(acc[r].y, mul(v.x, gk.y));
                        } else if constexpr ((P::im(k) >> r) & 1u) {
                            acc[r].x = sub(acc[r].x, mul(v.y, gk.y));
                            acc[r].y = add(acc[r].y, mul(v.y, gk.x));
                        } else {
                            acc[r] = O::vadd(acc[r], O::prod(v, gk));
                        }
                    }
                });
                // own rows of the gathered operand come from the site block
                if constexpr (k >= P::OWN && k < P::OWN + G) ui[k - P::OWN] = g[k - HF * NH];
            }
        });
    };
    auto mac_pat = [&](int pat, auto half_tag, const T (&g)[NH], const M* vs, T (&acc)[G],
                       T (&ui)[G]) {
        if constexpr (CPLX) {
            if (pat == 1)
                mac_half(PatTiMid{}, half_tag, g, vs, acc, ui);
            else if (pat == 2)
                mac_half(PatTiLo{}, half_tag, g, vs, acc, ui);
            else
                mac_half(PatTiHi{}, half_tag, g, vs, acc, ui);
        }
    };
    // generic group: quads of four columns, the next quad's gathers in flight while one is
    // multiplied; the value stream runs one value ahead of the products
    auto mac_generic = [&](const int4& h, const int* seg, const M* vseg, const Rows& q, T (&acc)[G],
                           T (&ui)[G]) {
        const int4* cs = reinterpret_cast<const int4*>(seg + h.x);
        const int nq = h.z >> 2;
        const M* vp = vseg + h.y;
        M vcur = *vp;
        auto mac = [&](int cw, const T& g) {
            const unsigned m = static_cast<unsigned>(cw) >> 28;
#pragma unroll
            for (int r = 0; r < G; ++r)
                if (m & (1u << r)) {
                    const M v = vcur;
                    ++vp;
                    vcur = *vp;
                    acc[r] = O::vadd(acc[r], O::prod(v, g));
                }
        };
        struct Quad {
            int4 c;
            T g[4];
        };
        auto load = [&](Quad& qd, int i) {
            qd.c = cs[i];
            qd.g[0] = ldgk(&inu[col_of(qd.c.x)]);
            qd.g[1] = ldgk(&inu[col_of(qd.c.y)]);
            qd.g[2] = ldgk(&inu[col_of(qd.c.z)]);
            qd.g[3] = ldgk(&inu[col_of(qd.c.w)]);
        };
        auto proc = [&](const Quad& qd) {
            mac(qd.c.x, qd.g[0]);
            mac(qd.c.y, qd.g[1]);
            mac(qd.c.z, qd.g[2]);
            mac(qd.c.w, qd.g[3]);
        };
        Quad qa, qb;
        if (nq > 0) load(qa, 0);
        for (int i = 0; i < nq; i += 2) {
            if (i + 1 < nq) load(qb, i + 1);
            proc(qa);
            if (i + 1 >= nq) break;
            if (i + 2 < nq) load(qa, i + 2);
            proc(qb);
        }
#pragma unroll
        for (int r = 0; r < G; ++r) ui[r] = ldgk(&inu[q.own[r] + halo * pitch]);
    };
    auto finish = [&](const Rows& q, const T (&acc)[G], const T (&ui)[G], const T (&wi)[G],
                      T (&xi)[G]) {
        T x0v[G];
#pragma unroll
        for (int r = 0; r < G; ++r) {
            x0v[r] = T{};
            if constexpr (kind_reads_x(KIND) && !CFD_GRP_X_EARLY) xi[r] = ldst(&X[q.own[r]]);
            if constexpr (DMODE == 2 && KIND != kStepStart2) x0v[r] = ldst(&X0[q.own[r]]);
        }
        if constexpr (SACC) {
            A dl[NDOT], dc[NDOT];
#pragma unroll
            for (int d = 0; d < NDOT; ++d) dl[d] = dc[d] = A{};
#pragma unroll
            for (int r = 0; r < G; ++r)
                if (q.ok[r])
                    step_epilogue<O, T, KIND, DMODE>(acc[r], ui[r], wi[r], xi[r], x0v[r], q.own[r], W,
                                                     X, X0, p.beta, coeff, c1, c2, dl, dc);
#pragma unroll
            for (int d = 0; d < NDOT; ++d) sacc[d * blockDim.x + t] = tadd(sacc[d * blockDim.x + t], dl[d]);
        } else {
#pragma unroll
            for (int r = 0; r < G; ++r)
                if (q.ok[r])
                    step_epilogue<O, T, KIND, DMODE>(acc[r], ui[r], wi[r], xi[r], x0v[r], q.own[r], W,
                                                     X, X0, p.beta, coeff, c1, c2, acc_d, comp_d);
        }
    };

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
    // tile schedule as step_tma_kernel: ORDER 0 persistent, CTA-strided (fixed CTA-to-tile
    // map: reproducible dot partials); ORDER 1 p.tile_a consecutive tiles per CTA, band order
    const int64_t tstride = ORDER == 0 ? static_cast<int64_t>(gridDim.x) : 1;
    int64_t tile = ORDER == 0 ? static_cast<int64_t>(blockIdx.x) : blockIdx.x * p.tile_a;
    const int64_t tend = ORDER == 0 ? ntiles : min(ntiles, tile + p.tile_a);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (t == 0 && tile < tend) issue(tile, 0);
    unsigned phases = 0u;
    for (int k = 0; tile < tend; ++k, tile += tstride) {
        const int buf = k & 1;
        if (tile + tstride >= tend) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        if (t == 0 && tile + tstride < tend) issue(tile + tstride, buf ^ 1);
        const int64_t tt = first_chunk(tile) / NCH;
        mbar_wait(&bars[buf], (phases >> buf) & 1u);
        phases ^= 1u << buf;
        const int* seg = cols_s + buf * gp.cap_c;
        const M* vseg = vals_s + buf * gp.cap_v;
        for (int it = 0; it < kTileGroups; it += R) {
            const int gi = it + rr;
            const int64_t rg = gp.tm.first_row(tt, gi);
            if (rg >= row1) continue;
            const int4 h = reinterpret_cast<const int4*>(seg)[gi];
            const Rows q = rows_of(rg);
            T acc[G], ui[G], wi[G], xi[G];
#pragma unroll
            for (int r = 0; r < G; ++r) {
                acc[r] = O::zero();
                ui[r] = T{};
            }
            load_w(q, wi, xi);
            if (h.w == 0) {
                mac_generic(h, seg, vseg, q, acc, ui);
            } else {
                // static pattern: every gather issued before the first product
                T gx[NH], gy[NH];
                gather_half(gx, gi, seg, 0);
                gather_half(gy, gi, seg, 1);
                const M* vs = vseg + h.y;
                mac_pat(h.w, std::integral_constant<int, 0>{}, gx, vs, acc, ui);
                mac_pat(h.w, std::integral_constant<int, 1>{}, gy, vs, acc, ui);
            }
            finish(q, acc, ui, wi, xi);
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

// CTA shape: up to 128 threads, R <= 16 groups per pass (a tile holds 16), one thread per
// 16-byte unit of a group's four rows; rows wider than 128 units run in column slabs
constexpr int kGroupSlabMax = 128;
inline Geometry group_geometry(int us) {
    Geometry g;
    g.US = us;
    int r = 1;
    while (r * 2 * us <= 128 && r * 2 <= kTileGroups) r *= 2;
    g.R = r;
    g.threads = r * us;
    return g;
}

// band tile order of a row-group launch (set_band_order): slices must be whole tiles
inline bool group_band_order(const Context& ctx, const Matrix& a, StepParams& p, size_t row_bytes,
                             int64_t tile_span) {
    set_band_order(ctx, a, p, kTileRows, row_bytes);
    if (p.band_tps != 0 && (p.band_plane_chunks % 2 != 0 || p.band_slice_chunks % 2 != 0 ||
                            (p.band_slice_chunks * 32) % tile_span != 0))
        p.band_tps = 0;
    return p.band_tps != 0;
}

inline const void* find_scaled_grouped(const Matrix& a, double s) {
    for (const auto& e : a.grp.scaled)
        if (e.first == s) return e.second->p;
    return nullptr;
}

// Launch the row-group kernel for s if it applies; false = nothing launched.
template <bool CPLX, class T, int KIND, int DMODE>
bool run_group(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch) {
    const Matrix& a = *s.a;
    const GroupedMatrix& gm = a.grp;
    constexpr int NDOT = dots_of(DMODE);
    using M = typename Ops<CPLX, T>::M;
    const int64_t nrows = s.row1 - s.row0;
    if (!ctx.grouped || ctx.kernel_variant != 1 || !gm.ok || nrows <= 0) return false;
    // launch ranges must be whole tiles (line groups of line-interleaved tiles)
    const int64_t tile_span = gm.il_line_rows ? gm.il_lines * gm.il_line_rows : kTileRows;
    if (s.row0 % tile_span != 0) return false;
    if (gm.il_line_rows && s.row1 % tile_span != 0) return false;
    const void* svals = s.alpha == 1.0 ? gm.vals.p : find_scaled_grouped(a, s.alpha);
    if (!svals) return false;
    const int slab = ctx.slab_units > 0 ? std::min(ctx.slab_units, kGroupSlabMax) : kGroupSlabMax;
    if (units > slab && NDOT > 0 && !s.final_launch) return false;
    // Default (CHEBFD_OPT_GROUPED = 1): only the launches that run in the band tile order,
    // i.e. dot-free steps on lattice operators whose z-planes exceed the L2 budget (C4, C3 at
    // n_b = 256: 7-17 % faster than the SELL kernel).  Where the planes are L2-resident the
    // SELL kernel's 16 warps/SM win (C2: 0.50 against 0.62 ms per step), measured with
    // tools/group_exp.py.
    if (ctx.grouped == 1) {
        if (DMODE != 0 || ctx.tiles_per_cta <= 0) return false;
        StepParams probe{};
        probe.row0 = s.row0;
        probe.row1 = s.row1;
        if (!group_band_order(ctx, a, probe, static_cast<size_t>(std::min(slab, units)) * sizeof(T),
                              tile_span))
            return false;
    }
    int used_total = 0;
    for (int u0 = 0; u0 < units; u0 += slab) {
        const int us = std::min(slab, units - u0);
        const Geometry g = group_geometry(us);
        GroupParams gp{};
        gp.tile_cptr = gm.tile_cptr.as<int64_t>();
        gp.tile_vptr = gm.tile_vptr.as<int64_t>();
        gp.cols = gm.cols.as<int>();
        gp.vals = svals;
        gp.cap_c = gm.max_tile_cols;
        gp.cap_v = gm.max_tile_vals + 2;  // the value stream reads one ahead
        gp.tm = tilemap_of(gm);
        size_t ring = 2 * static_cast<size_t>(gp.cap_c) * sizeof(int) +
                      2 * static_cast<size_t>(gp.cap_v) * sizeof(M);
        if (NDOT > 0 && DMODE != 1) ring += NDOT * static_cast<size_t>(g.threads) * sizeof(T);
        const size_t smem = std::max(NDOT * static_cast<size_t>(g.threads) * sizeof(T), ring);
        if (smem > 200 * 1024) return false;
        auto kernel = step_group_kernel<CPLX, T, KIND, DMODE, 0>;
        StepParams p{};
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
        p.dots_row_stride = static_cast<int64_t>(units) * Ops<CPLX, T>::kCols;
        p.tr = kTileRows;
        p.band_tps = 0;
        p.tile_a = 1;
        const int64_t need = (((s.row1 + 31) >> 5) - (s.row0 >> 5) + 1) / 2;
        bool band = false;
        if constexpr (DMODE == 0) {
            if (ctx.tiles_per_cta > 0)
                band = group_band_order(ctx, a, p, static_cast<size_t>(us) * sizeof(T), tile_span);
        }
        if (band) kernel = step_group_kernel<CPLX, T, KIND, DMODE, DMODE == 0 ? 1 : 0>;
        static thread_local std::map<std::pair<const void*, int>, size_t> attr_set;
        auto& cur = attr_set[std::make_pair(reinterpret_cast<const void*>(kernel), ctx.device)];
        if (smem > 48 * 1024 && cur < smem) {
            CFD_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem)));
            cur = smem;
        }
        int grid;
        if (band) {
            const int64_t tpc = ctx.tiles_per_cta;
            grid = static_cast<int>((need + tpc - 1) / tpc);
            p.tile_a = tpc;
            ++ctx.band_launches;
        } else {
            static thread_local std::map<std::tuple<const void*, int, size_t, int>, int> occ_cache;
            auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), g.threads, smem, ctx.device);
            auto it = occ_cache.find(key);
            const int maxb = it != occ_cache.end()
                                 ? it->second
                                 : (occ_cache[key] = max_blocks_for(kernel, g.threads, smem, ctx.num_sms));
            grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, maxb)));
        }
        if (NDOT > 0) {
            const size_t need_bytes =
                static_cast<size_t>(reduce_rows_needed(s.partial_base + grid)) * NDOT * us * sizeof(T);
            ctx.partials.ensure(std::max<size_t>(need_bytes, 1 << 20));
            ctx.counter.ensure(4096);
        }
        p.partials = ctx.partials.p;
        p.part_base = s.partial_base;
        p.nparts = s.partial_base + grid;
        p.final_launch = s.final_launch ? 1 : 0;
        p.counter = ctx.counter.as<unsigned>();
        const bool pdl = s.pdl_ok && ctx.pdl == 2;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(grid));
        cfg.blockDim = dim3(static_cast<unsigned>(g.threads));
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CFD_CUDA(cudaLaunchKernelEx(&cfg, kernel, p, gp));
        CFD_CUDA(cudaGetLastError());
        ctx.launches++;
        ctx.group_launches++;
        used_total = grid;
    }
    if (s.grid_used) *s.grid_used = used_total;
    return true;
}

template <bool CPLX, class T>
bool dispatch_group(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch) {
    switch (s.kind_step) {
        case kStepSpmmvm:
            if (s.dots_mode == 3) return run_group<CPLX, T, kStepSpmmvm, 3>(ctx, s, st, units, pitch);
            if (s.dots_mode == 4) return run_group<CPLX, T, kStepSpmmvm, 4>(ctx, s, st, units, pitch);
            return run_group<CPLX, T, kStepSpmmvm, 0>(ctx, s, st, units, pitch);
        case kStepStart2:
            if (s.dots_mode == 2) return run_group<CPLX, T, kStepStart2, 2>(ctx, s, st, units, pitch);
            if (s.dots_mode == 4) return run_group<CPLX, T, kStepStart2, 4>(ctx, s, st, units, pitch);
            return run_group<CPLX, T, kStepStart2, 0>(ctx, s, st, units, pitch);
        case kStepFused:
            if (s.dots_mode == 1) return run_group<CPLX, T, kStepFused, 1>(ctx, s, st, units, pitch);
            if (s.dots_mode == 2) return run_group<CPLX, T, kStepFused, 2>(ctx, s, st, units, pitch);
            if (s.dots_mode == 4) return run_group<CPLX, T, kStepFused, 4>(ctx, s, st, units, pitch);
            return run_group<CPLX, T, kStepFused, 0>(ctx, s, st, units, pitch);
        case kStepFusedX2:
            if (s.dots_mode == 2) return run_group<CPLX, T, kStepFusedX2, 2>(ctx, s, st, units, pitch);
            if (s.dots_mode == 0) return run_group<CPLX, T, kStepFusedX2, 0>(ctx, s, st, units, pitch);
            break;
        case kStepFusedX3:
            if (s.dots_mode == 2) return run_group<CPLX, T, kStepFusedX3, 2>(ctx, s, st, units, pitch);
            if (s.dots_mode == 0) return run_group<CPLX, T, kStepFusedX3, 0>(ctx, s, st, units, pitch);
            break;
        case kStepRecur:
            if (s.dots_mode == 2) return run_group<CPLX, T, kStepRecur, 2>(ctx, s, st, units, pitch);
            if (s.dots_mode == 4) return run_group<CPLX, T, kStepRecur, 4>(ctx, s, st, units, pitch);
            if (s.dots_mode == 5) return run_group<CPLX, T, kStepRecur, 5>(ctx, s, st, units, pitch);
            if (s.dots_mode == 6) return run_group<CPLX, T, kStepRecur, 6>(ctx, s, st, units, pitch);
            return run_group<CPLX, T, kStepRecur, 0>(ctx, s, st, units, pitch);
    }
    return false;
}

}  // namespace
}  // namespace cfd
