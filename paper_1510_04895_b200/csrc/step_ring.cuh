// Site-ring step kernel (sm_100a): a warp-specialised Chebyshev step for topological-insulator
// lattice operators (complex blocks of 32 or 64 units per row / column slab).
//
// Why: the row-group kernel (step_group.cuh) gathers a site's 24 neighbour rows through the
// L1 with 255 registers per thread -- 8 warps per SM, whose loads and FP64 work do not
// overlap, and ~22 KB per site crossing the L2 -> SM path (L1 hit rate 21 %).  Here the
// gathered operand never touches a register before it is multiplied:
//
//   * a CTA owns a strip of SY = 4 adjacent lattice lines of one z-plane and marches along x;
//   * one PRODUCER warp copies, per x-column, the strip's site blocks (SY + 2 sites of the
//     own plane: the strip and its y -+ 1 halo sites) and the z -+ 1 rows + matrix values of
//     the column's sites into shared-memory rings with TMA bulk copies
//     (cp.async.bulk ... mbarrier::complete_tx), several columns ahead;
//   * CONSUMER warps (one 16-byte unit of a site's four rows per thread, as the row-group
//     kernel) read every operand from shared memory: x -+ 1 neighbours are the neighbouring
//     ring slots, y -+ 1 neighbours the neighbouring lines' slots, so a site block crosses
//     L2 -> SM once per strip (+ halo) instead of once per referencing site:
//     ~10.7 KB per site instead of ~22 KB;
//   * full / empty mbarriers per ring slot; no __syncthreads after the roles split.
//
// Each row still meets its entries in CSR order with the reference's roundings (the static
// site patterns of group_patterns.hpp; x / y wrap sites take a generic path that gathers
// from global memory), so W and X are bit-identical to the other step kernels.
//
// The producer's addresses come from a per-site plan built with the grouped form
// (group.cu build_ring_plan): the z -+ 1 row indices (extended rows, so compact halos and
// rank boundaries need nothing special), the site's value offset and pattern id.  x / y
// neighbours of static sites are checked there to be the lattice neighbours.
#pragma once
#include <cuda.h>

#include <utility>

#include "group_patterns.hpp"
#include "step_kernels.cuh"

namespace cfd {
namespace {

#ifndef CFD_RING_PREFETCH
#define CFD_RING_PREFETCH 2  // columns ahead the consumers' W / X rows are prefetched into the L2
#endif
#ifndef CFD_RING_ROTATE
#define CFD_RING_ROTATE 1
#endif
#ifndef CFD_RING_SHARE
#define CFD_RING_SHARE 1  // row pairs share the products of an x / y neighbour column (PatBase::pair_col)
#endif
constexpr int kRingSY = 4;         // lattice lines per strip
constexpr int kRingMaxDepth = 8;   // ring slots (each ring)

struct RingParams {
    const int4* plan;   // two int4 per site (group.cu)
    const int* cols;    // grouped columns (generic sites)
    const void* vals;   // grouped values pre-multiplied by alpha
    int lx, ly;         // sites per line, lines per plane
    int planes;         // planes of this launch
    int segx, nseg;     // x-columns per CTA, segments per line
    int spb;            // strips per band (band order of the grid)
    int nbands, order;  // bands per plane; 0: x segments fastest, 1: x segments slowest
    int no, nz;         // ring depths: own-plane columns, z / value stages
    int full;           // 1: the slab is the whole row (a site's four rows are one 1D copy)
    int tmap;           // 1: tensor-map copies (RingMaps): whole sites / row pairs for any slab
};

// per pattern, the (alpha-scaled) real or imaginary part of every purely real / imaginary
// matrix value that is the same at all static sites (GroupedMatrix::ring_consts); a kernel
// parameter, so the products take it as a constant-bank operand: no load, no register
struct RingConsts {
    double v[3][kRingMaxVals];
};

template <class F, int... I>
__device__ __forceinline__ void ring_for_impl(F&& f, std::integer_sequence<int, I...>) {
    (f(std::integral_constant<int, I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void ring_for(F&& f) {
    ring_for_impl(f, std::make_integer_sequence<int, N>{});
}

__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, unsigned bytes,
                                                 uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
        "[%3], %4;\n" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
// Tensor-map TMA (cp.async.bulk.tensor.2d, UTMALDG): the gathered block as a 2D tensor
// [extended rows][doubles of a row]; a box is R rows x one slab of columns, so a site's four
// rows (or a z -+ 1 row pair) of any column slab travel as ONE copy whatever the row pitch.
struct RingMaps {
    CUtensorMap m4, m2, m1;  // boxes of 4, 2 and 1 rows
};
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* tm, int c0, int c1,
                                                 uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
using TensorMapEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                       const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                       const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                       CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
// cuTensorMapEncodeTiled through the runtime (the library does not link libcuda); null if absent
inline TensorMapEncodeFn tensor_map_encoder() {
    static TensorMapEncodeFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<TensorMapEncodeFn>(f);
    }();
    return fn;
}
// maps over the block at `base` (ext_rows rows of `pitch` 16-byte units), boxes of us units
inline bool make_ring_maps(RingMaps& m, const void* base, int64_t ext_rows, int pitch, int us) {
    TensorMapEncodeFn enc = tensor_map_encoder();
    if (!enc) return false;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(pitch) * 2, static_cast<cuuint64_t>(ext_rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch) * 16};
    const cuuint32_t estr[2] = {1, 1};
    CUtensorMap* maps[3] = {&m.m4, &m.m2, &m.m1};
    const cuuint32_t rows[3] = {4, 2, 1};
    for (int i = 0; i < 3; ++i) {
        const cuuint32_t box[2] = {static_cast<cuuint32_t>(us) * 2, rows[i]};
        if (enc(maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box,
                estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    return true;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// shared-memory bases of a site's operand classes (unit offset included)
struct RingBases {
    const unsigned char *zlo, *ym, *xm, *own, *xp, *yp, *zhi;
};

// operand k of pattern P: columns run z-1 | y-1 | x-1 | site | x+1 | y+1 | z+1
template <class P, int K, int RB>
__device__ __forceinline__ double2 ring_operand(const RingBases& b) {
    constexpr int ZLO = P::OWN - 8;  // z-1 columns in front (2 or 0)
    constexpr int q = K - ZLO;
    const unsigned char* a;
    if constexpr (K < ZLO)
        a = b.zlo + K * RB;
    else if constexpr (q < 4)
        a = b.ym + q * RB;
    else if constexpr (q < 8)
        a = b.xm + (q - 4) * RB;
    else if constexpr (q < 12)
        a = b.own + (q - 8) * RB;
    else if constexpr (q < 16)
        a = b.xp + (q - 12) * RB;
    else if constexpr (q < 20)
        a = b.yp + (q - 16) * RB;
    else
        a = b.zhi + (q - 20) * RB;
    return *reinterpret_cast<const double2*>(a);
}

// products of the rows R0 .. R0 + RS - 1 of a static-pattern site: only the operands those
// rows (or their own-row terms) need are read
template <class P, int RB, int R0, int RS, bool CV>
__device__ __forceinline__ void ring_mac(const RingBases& b, const double2* vs, const RingConsts& cc,
                                         double2 (&acc)[RS], double2 (&ui)[RS]) {
    using O = Ops<true, double2>;
    constexpr unsigned SUB = ((1u << RS) - 1u) << R0;
    ring_for<P::NC>([&](auto kt) {
        constexpr int k = decltype(kt)::value;
        constexpr bool own = k >= P::OWN + R0 && k < P::OWN + R0 + RS;
        constexpr bool shared_pair = CFD_RING_SHARE != 0 && CV && RS == 2 && P::pair_col(k) && (P::m(k) & SUB) == SUB;
        if constexpr (shared_pair) {
            // both rows of this thread's pair read column k with values +-v / +-iv of one
            // magnitude: the two products v g_r, v g_i serve both rows
            static_assert((((P::re(k) | P::im(k)) & SUB) == SUB) && !own, "pair column: purely real / imaginary values");
            const double2 gk = ring_operand<P, k, RB>(b);
            const double v = cc.v[P::ID][P::voff(k, R0)];
            const double px = mul(v, gk.x), py = mul(v, gk.y);
            if constexpr ((P::re(k) >> R0) & 1u) {
                acc[0].x = add(acc[0].x, px);
                acc[0].y = add(acc[0].y, py);
            } else {
                acc[0].x = sub(acc[0].x, py);
                acc[0].y = add(acc[0].y, px);
            }
            constexpr bool neg = P::pair_neg(k);
            if constexpr ((P::re(k) >> (R0 + 1)) & 1u) {
                acc[1].x = neg ? sub(acc[1].x, px) : add(acc[1].x, px);
                acc[1].y = neg ? sub(acc[1].y, py) : add(acc[1].y, py);
            } else {
                acc[1].x = neg ? add(acc[1].x, py) : sub(acc[1].x, py);
                acc[1].y = neg ? sub(acc[1].y, px) : add(acc[1].y, px);
            }
        } else if constexpr ((P::m(k) & SUB) != 0u || own) {
            const double2 gk = ring_operand<P, k, RB>(b);
            ring_for<RS>([&](auto rt) {
                constexpr int r = R0 + decltype(rt)::value;
                constexpr int a = decltype(rt)::value;
                if constexpr ((P::m(k) >> r) & 1u) {
                    constexpr bool cv = CV && k != P::OWN + r;  // not the site's diagonal entry
                    if constexpr ((P::re(k) >> r) & 1u) {
                        double v;
                        if constexpr (cv)
                            v = cc.v[P::ID][P::voff(k, r)];
                        else
                            v = vs[P::voff(k, r)].x;
                        acc[a].x = add(acc[a].x, mul(v, gk.x));
                        acc[a].y = add(acc[a].y, mul(v, gk.y));
                    } else if constexpr ((P::im(k) >> r) & 1u) {
                        double v;
                        if constexpr (cv)
                            v = cc.v[P::ID][P::voff(k, r)];
                        else
                            v = vs[P::voff(k, r)].y;
                        acc[a].x = sub(acc[a].x, mul(v, gk.y));
                        acc[a].y = add(acc[a].y, mul(v, gk.x));
                    } else {
                        acc[a] = O::vadd(acc[a], O::prod(vs[P::voff(k, r)], gk));
                    }
                }
            });
            if constexpr (own) ui[k - P::OWN - R0] = gk;
        }
    });
}

// RS rows of a site per consumer thread (4, 2 or 1): 4 / RS consumer groups share a site's
// operands in shared memory, which multiplies the resident consumer warps -- the FP64
// chains of 8 warps per SM do not fill the issue slots (ncu: issue 35 % busy, stalls on
// fixed-latency dependencies)
//
// DMODE 4 / 5 / 6 (V_n-only steps of a moment-collecting filter or a KPM run): the raw moment
// sums of step_epilogue from the consumers' registers; per-thread sums over the CTA's columns
// in order -> CTA partials -> grid_reduce in CTA index order (bitwise reproducible).
template <int KIND, int US, int RS, bool CV, int SY = kRingSY, int DMODE = 0>
__global__ void __launch_bounds__((kGroupRows / RS) * SY * US + 64, (US == 32 && RS >= 2) ? 2 : 1)
    step_ring_kernel(const StepParams p, const RingParams rp, const __grid_constant__ RingConsts cc,
                     const __grid_constant__ RingMaps tm) {
    using T = double2;
    using O = Ops<true, double2>;
    using M = double2;
    constexpr int G = kGroupRows;
    constexpr int NG = G / RS;                      // consumer groups
    constexpr int RB = US * 16;                     // bytes of a row (slab)
    constexpr int OS = (SY + 2) * G * RB;           // own-plane column slot
    constexpr int VB = kRingMaxVals * 16;           // value bytes per site
    constexpr int ZS = SY * G * RB + SY * VB;       // z-row + value stage
    constexpr int NCT = SY * US;                    // consumer threads per group
    constexpr int NCW = NG * NCT / 32;              // consumer warps
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[4 * kRingMaxDepth];
    uint64_t* full_o = bars;
    uint64_t* empty_o = bars + kRingMaxDepth;
    uint64_t* full_z = bars + 2 * kRingMaxDepth;
    uint64_t* empty_z = bars + 3 * kRingMaxDepth;
    constexpr int NDOT = dots_of(DMODE);
    static_assert(NDOT == 0 || (KIND == kStepRecur && DMODE >= 4), "ring dots: moment sums of V_n-only steps");
    double acc_d[NDOT > 0 ? NDOT : 1] = {}, comp_d[NDOT > 0 ? NDOT : 1] = {};
    const int t = threadIdx.x;
    const int no = rp.no, nz = rp.nz;
    unsigned char* oring = smem_raw;
    unsigned char* zring = oring + static_cast<size_t>(no) * OS;
    int4* plan_s = reinterpret_cast<int4*>(zring + static_cast<size_t>(nz) * ZS);

    // CTA -> (band of strips, plane, strip in the band, x segment): planes innermost over a
    // band, so the z -+ 1 rows a strip reads were own rows of a CTA a band slice earlier
    unsigned idx = blockIdx.x;
    int q, sb, z, band;
    if (rp.order == 0) {
        q = static_cast<int>(idx % static_cast<unsigned>(rp.nseg));
        idx /= static_cast<unsigned>(rp.nseg);
        sb = static_cast<int>(idx % static_cast<unsigned>(rp.spb));
        idx /= static_cast<unsigned>(rp.spb);
        z = static_cast<int>(idx % static_cast<unsigned>(rp.planes));
        band = static_cast<int>(idx / static_cast<unsigned>(rp.planes));
    } else if (rp.order == 2) {
        // planes fastest, then strips, x segment slowest: a CTA's z neighbours are its
        // neighbours in launch order and its y neighbours `planes` CTAs away, so a wave of
        // CTAs is a compact (strips x planes) brick marching along x in lockstep and a wave
        // boundary separates one plane pair and `planes` strip pairs at most
        z = static_cast<int>(idx % static_cast<unsigned>(rp.planes));
        idx /= static_cast<unsigned>(rp.planes);
        sb = static_cast<int>(idx % static_cast<unsigned>(rp.spb));
        q = static_cast<int>(idx / static_cast<unsigned>(rp.spb));
        band = 0;

    } else {
        // x segment slowest: a wave of CTAs is (all planes) x (spb adjacent strips) of one x
        // segment marching in lockstep, so the strips' y -+ 1 halo lines and z -+ 1 rows are
        // being read by their owners at the same time (one DRAM read, L2 hits for the rest)
        sb = static_cast<int>(idx % static_cast<unsigned>(rp.spb));
        idx /= static_cast<unsigned>(rp.spb);
        z = static_cast<int>(idx % static_cast<unsigned>(rp.planes));
        idx /= static_cast<unsigned>(rp.planes);
        band = static_cast<int>(idx % static_cast<unsigned>(rp.nbands));
        q = static_cast<int>(idx / static_cast<unsigned>(rp.nbands));
    }
    const int lx = rp.lx, ly = rp.ly, segx = rp.segx;
    // the plane's last strip first: the first and the last strip hold the y-wrap (or open-edge)
    // lines, whose sites run the generic path -- the slowest CTAs then start a sweep's first
    // wave instead of forming the kernel's tail (C4: filter 5.97 -> 5.80 ms per step, fused step
    // 0.95 -> 0.98 of measured HBM); strips 127 and 0 are y neighbours, so bands stay compact
    int strip = band * rp.spb + sb;
#if CFD_RING_ROTATE
    strip = strip == 0 ? rp.spb * rp.nbands - 1 : strip - 1;
#endif
    const int y0 = strip * SY;
    const int xa = q * segx;
    const int xb = min(lx, xa + segx);
    const int jlo = xa > 0 ? xa - 1 : xa;  // own-plane columns [jlo, jhi): the segment + aprons
    const int jhi = xb < lx ? xb + 1 : xb;
    // owned site index of (x = 0, line y0) of this plane
    const int64_t site0 = (p.row0 >> 2) + (static_cast<int64_t>(z) * ly + y0) * lx;

    // the segment's plan -> shared memory (matrix data: may precede the previous kernel's end)
    {
        const int n2 = 2 * (xb - xa);
        for (int i = t; i < SY * 2 * segx; i += blockDim.x) {
            const int l = i / (2 * segx), r = i - l * 2 * segx;
            if (r < n2) plan_s[i] = __ldg(&rp.plan[2 * (site0 + static_cast<int64_t>(l) * lx + xa) + r]);
        }
    }
    if (t == 0) {
        for (int i = 0; i < no; ++i) {
            mbar_init(&full_o[i], 1);
            mbar_init(&empty_o[i], NCW);
        }
        for (int i = 0; i < nz; ++i) {
            mbar_init(&full_z[i], 2);  // one arrival per producer warp
            mbar_init(&empty_z[i], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int pitch = p.pitch;

    if (t >= NG * NCT) {
        // ============================== producer warps ===============================
        // Two warps, because issuing a bulk copy costs ~90 cycles of a warp (the lanes'
        // operands move to uniform registers one copy at a time): warp A feeds the
        // own-plane ring and the sites' matrix values, warp B the z -+ 1 rows.
        const int pw = (t - NG * NCT) >> 5;
        const int lane = t & 31;
        const T* inb = static_cast<const T*>(p.in) + p.u_off;
        const uint64_t pol_keep = l2_make_policy(1);
        const int K = jhi - jlo;
        if (pw == 0) {
            const M* gvals = static_cast<const M*>(rp.vals);
            const uint64_t pol_stream = l2_make_policy(2);
            // own-plane copies of this lane: site slot ss (row rr of it unless whole sites)
            int ss, rr;
            unsigned obytes;
            bool oact;
            if (rp.full || rp.tmap) {
                ss = lane;
                rr = 0;
                obytes = G * RB;
                oact = lane < SY + 2;
            } else {
                ss = lane >> 2;
                rr = lane & 3;
                obytes = RB;
                oact = lane < G * (SY + 2);
            }
            {
                const int y = y0 + ss - 1;
                oact = oact && y >= 0 && y < ly;
            }
            const bool oin = ss >= 1 && ss <= SY;  // a strip line (aprons copy only these)
            const int64_t erow0 = p.halo_lo + G * (site0 + static_cast<int64_t>(ss - 1) * lx) + rr;
            unsigned char* odst0 = oring + (ss * G + rr) * RB;
            int oslot = 0, opar = 1;  // empty-barrier parity of the slot's previous use
            int zslot = 0, zpar = 1;
            for (int k = 0; k <= K; ++k) {
                if (k < K) {
                    const int j = jlo + k;
                    if (k >= no) mbar_wait(&empty_o[oslot], opar);
                    const bool act = oact && ((j >= xa && j < xb) || oin);
                    const unsigned total = __reduce_add_sync(0xffffffffu, act ? obytes : 0u);
                    if (lane == 0) mbar_arrive_expect_tx(&full_o[oslot], total);
                    __syncwarp();
                    if (act) {
                        if (rp.tmap)
                            tma_load_2d_hint(odst0 + static_cast<size_t>(oslot) * OS, &tm.m4, p.u_off * 2,
                                             static_cast<int>(erow0 + static_cast<int64_t>(G) * j),
                                             &full_o[oslot], pol_keep);
                        else
                            tma_load_1d_hint(odst0 + static_cast<size_t>(oslot) * OS,
                                             inb + (erow0 + static_cast<int64_t>(G) * j) * pitch, obytes,
                                             &full_o[oslot], pol_keep);
                    }
                    if (++oslot == no) {
                        oslot = 0;
                        opar ^= 1;
                    }
                }
                const int c = jlo + k - 1;
                if (c >= xa && c < xb) {  // the column's matrix values (one copy per site)
                    const int kz = c - xa;
                    if (kz >= nz) mbar_wait(&empty_z[zslot], zpar);
                    unsigned bytes = 0;
                    const void* src = nullptr;
                    unsigned char* dst = zring + static_cast<size_t>(zslot) * ZS + SY * G * RB + lane * VB;
                    if (lane < SY) {
                        const int4 b = plan_s[(lane * segx + kz) * 2 + 1];
                        const int64_t voff = static_cast<int64_t>(static_cast<unsigned>(b.x)) |
                                             (static_cast<int64_t>(b.y) << 32);
                        // constants cover the static sites' off-diagonal values: their four
                        // diagonal entries sit inside the first (OWN + 4) columns' values
                        bytes = static_cast<unsigned>(b.w) * 16u;
                        src = gvals + voff;
                    }
                    const unsigned total = __reduce_add_sync(0xffffffffu, bytes);
                    if (lane == 0) mbar_arrive_expect_tx(&full_z[zslot], total);
                    __syncwarp();
                    if (bytes) tma_load_1d_hint(dst, src, bytes, &full_z[zslot], pol_stream);
                    if (++zslot == nz) {
                        zslot = 0;
                        zpar ^= 1;
                    }
                }
            }
        } else {
            int zslot = 0, zpar = 1;
            for (int c = xa; c < xb; ++c) {
                const int kz = c - xa;
                if (kz >= nz) mbar_wait(&empty_z[zslot], zpar);
                unsigned bytes = 0;
                const void* src = nullptr;
                int zrow = 0;
                unsigned char* dst = zring + static_cast<size_t>(zslot) * ZS;
                if (lane < G * SY) {
                    const int l = lane >> 2, w = lane & 3;
                    const int4 a = plan_s[(l * segx + kz) * 2];
                    const int4 b = plan_s[(l * segx + kz) * 2 + 1];
                    const int row = w == 0 ? a.x : (w == 1 ? a.y : (w == 2 ? a.z : a.w));
                    const int prev = w == 1 ? a.x : (w == 3 ? a.z : -2);   // the pair's first row
                    const int next = w == 0 ? a.y : (w == 2 ? a.w : -2);   // the pair's second row
                    if (b.z != 0 && row >= 0) {
                        // adjacent rows of a pair (whole-row slabs) travel as one copy
                        const bool pairs = rp.full || rp.tmap;
                        const bool merged_away = pairs && prev >= 0 && row == prev + 1;
                        const bool merges = pairs && next == row + 1;
                        if (!merged_away) {
                            bytes = merges ? 2 * RB : RB;
                            src = inb + static_cast<int64_t>(row) * pitch;
                            zrow = row;
                            dst += (l * G + w) * RB;
                        }
                    }
                }
                const unsigned total = __reduce_add_sync(0xffffffffu, bytes);
                if (lane == 0) mbar_arrive_expect_tx(&full_z[zslot], total);
                __syncwarp();
                if (bytes) {
                    if (rp.tmap)
                        tma_load_2d_hint(dst, bytes == RB ? &tm.m1 : &tm.m2, p.u_off * 2, zrow,
                                         &full_z[zslot], pol_keep);
                    else
                        tma_load_1d_hint(dst, src, bytes, &full_z[zslot], pol_keep);
                }
                if (++zslot == nz) {
                    zslot = 0;
                    zpar ^= 1;
                }
            }
        }
    } else {
        // ================================ consumer warps ================================
        const int grp = t / NCT;
        const int tt = t - grp * NCT;
        const int l = tt / US, u = tt - l * US;
        const int cu = p.u_off + u;
        const bool lane0 = (t & 31) == 0;
        const T* __restrict__ inu = static_cast<const T*>(p.in) + cu;
        T* __restrict__ W = static_cast<T*>(p.w) + cu;
        T* __restrict__ X = static_cast<T*>(p.x) + cu;
        double coeff = p.c0, c1 = p.c1, c2 = p.c2;
        if (kind_fused(KIND) && p.coeff_dev) coeff = p.coeff_dev[p.coeff_index];
        if ((KIND == kStepFusedX2 || KIND == kStepFusedX3) && p.coeff_dev) c1 = p.coeff_dev[p.coeff_index - 1];
        if (KIND == kStepFusedX3 && p.coeff_dev) c2 = p.coeff_dev[p.coeff_index - 2];
        const uint64_t pol_stream = l2_make_policy(2);

        auto consume = [&](auto r0_tag) {
            constexpr int R0 = decltype(r0_tag)::value;
            // ring positions, advanced per column (no divisions in the loop)
            int so_m = no - 1, so_c = 0, so_p = 1 % no;    // slots of columns c - 1, c, c + 1
            if (xa > jlo) {
                so_m = 0;
                so_c = 1 % no;
                so_p = 2 % no;
            }
            int wslot = 0, wpar = 0, kw = 0;  // next own-plane column to wait for
            int zslot = 0, zpar = 0;
            const int64_t rg0 = G * (site0 + static_cast<int64_t>(l) * lx) + R0;
            // the own rows of the current column as running pointers (a column ahead = colstep
            // elements): recomputing (row) * pitch per access cost ~45 of the ~250 instructions
            // a warp spends on a column
            const int64_t colstep = static_cast<int64_t>(G) * pitch;
            T* wrow[RS];
            // X's rows sit at a launch-uniform distance from W's (no second pointer set)
            const int64_t xdelta = static_cast<T*>(p.x) - static_cast<T*>(p.w);
#pragma unroll
            for (int r = 0; r < RS; ++r) wrow[r] = W + (rg0 + static_cast<int64_t>(G) * xa + r) * pitch;
            auto load_rows = [&](T (&wv)[RS], T (&xv)[RS]) {
#pragma unroll
                for (int r = 0; r < RS; ++r) {
                    wv[r] = xv[r] = T{};
                    if constexpr (kind_reads_w(KIND)) wv[r] = lds_pol(wrow[r], pol_stream);
                    if constexpr (kind_reads_x(KIND)) xv[r] = lds_pol(wrow[r] + xdelta, pol_stream);
                }
            };
            // own-row streams (W, X): loaded at the top of the column's step and consumed in
            // its epilogue -- a whole step later -- after an L2 prefetch kPre columns ahead.
            // (Handing a next-column register buffer over at the end of a step stalled on
            // the loads in flight: 23 % of the ncu samples.)
            constexpr int kPre = CFD_RING_PREFETCH;
            auto prefetch_rows = [&](int ahead) {  // the own rows `ahead` columns ahead
#pragma unroll
                for (int r = 0; r < RS; ++r) {
                    if constexpr (kind_reads_w(KIND))
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(wrow[r] + ahead * colstep));
                    if constexpr (kind_reads_x(KIND))
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(wrow[r] + xdelta + ahead * colstep));
                }
            };
            if constexpr (kPre > 0) {
#pragma unroll
                for (int i = 1; i < kPre; ++i)
                    if (xa + i < xb) prefetch_rows(i);
            }
            for (int c = xa; c < xb; ++c) {
                const int kz = c - xa;
                const int4 pb = plan_s[(l * segx + kz) * 2 + 1];
                const int pat = pb.z;
                // static sites load their own rows now (consumed a whole step later); generic
                // sites after their gathers, whose registers they would otherwise take
                T wi[RS], xi[RS];
                if (pat != 0) load_rows(wi, xi);
                if constexpr (kPre > 0) {
                    if (c + kPre < xb) prefetch_rows(kPre);
                }
                const int need = min(c + 1, jhi - 1) - jlo;
                while (kw <= need) {
                    mbar_wait(&full_o[wslot], wpar);
                    ++kw;
                    if (++wslot == no) {
                        wslot = 0;
                        wpar ^= 1;
                    }
                }
                mbar_wait(&full_z[zslot], zpar);
                const unsigned char* oc = oring + static_cast<size_t>(so_c) * OS + u * 16;
                const unsigned char* om = oring + static_cast<size_t>(so_m) * OS + u * 16;
                const unsigned char* op = oring + static_cast<size_t>(so_p) * OS + u * 16;
                const unsigned char* zb = zring + static_cast<size_t>(zslot) * ZS;
                const M* vs = reinterpret_cast<const M*>(zb + SY * G * RB + l * VB);
                RingBases b;
                b.ym = oc + l * (G * RB);
                b.own = oc + (l + 1) * (G * RB);
                b.yp = oc + (l + 2) * (G * RB);
                b.xm = om + (l + 1) * (G * RB);
                b.xp = op + (l + 1) * (G * RB);
                b.zlo = zb + l * (G * RB) + u * 16;
                b.zhi = b.zlo + 2 * RB;
                T acc[RS], ui[RS];
#pragma unroll
                for (int r = 0; r < RS; ++r) acc[r] = O::zero();
                if (pat == 1) {
                    ring_mac<PatTiMid, RB, R0, RS, CV>(b, vs, cc, acc, ui);
                } else if (pat == 2) {
                    ring_mac<PatTiLo, RB, R0, RS, CV>(b, vs, cc, acc, ui);
                } else if (pat == 3) {
                    ring_mac<PatTiHi, RB, R0, RS, CV>(b, vs, cc, acc, ui);
                } else {
                    // generic site (x / y wrap, open edges): merged columns gathered from
                    // global memory; a column's values follow its set rows in increasing order
                    const int4 pa = plan_s[(l * segx + kz) * 2];
                    const int64_t coff = static_cast<int64_t>(static_cast<unsigned>(pa.x)) |
                                         (static_cast<int64_t>(pa.y) << 32);
                    const int* cl = rp.cols + coff;
                    const int n = pa.z;
                    constexpr unsigned SUB = ((1u << RS) - 1u) << R0;
                    int vi = 0;
                    // batches of eight columns: their gathers are all in flight before the
                    // first product (whole lines of such sites sit on the y wrap: two strips
                    // per plane run at this path's speed)
                    const int4* cl4 = reinterpret_cast<const int4*>(cl);
                    for (int k0 = 0; k0 < n; k0 += 8) {
                        const int4 ca = __ldg(cl4 + (k0 >> 2));
                        const int4 cb = k0 + 4 < n ? __ldg(cl4 + (k0 >> 2) + 1) : make_int4(0, 0, 0, 0);
                        const unsigned cw[8] = {static_cast<unsigned>(ca.x), static_cast<unsigned>(ca.y),
                                                static_cast<unsigned>(ca.z), static_cast<unsigned>(ca.w),
                                                static_cast<unsigned>(cb.x), static_cast<unsigned>(cb.y),
                                                static_cast<unsigned>(cb.z), static_cast<unsigned>(cb.w)};
                        T g[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            g[j] = T{};
                            if ((cw[j] >> 28) & SUB)
                                g[j] = ldg(&inu[static_cast<int64_t>(cw[j] & 0x0FFFFFFFu) * pitch]);
                        }
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const unsigned m = cw[j] >> 28;
#pragma unroll
                            for (int r = 0; r < RS; ++r)
                                if (m & (1u << (R0 + r)))
                                    acc[r] = O::vadd(
                                        acc[r], O::prod(vs[vi + __popc(m & ((1u << (R0 + r)) - 1u))], g[j]));
                            vi += __popc(m);
                        }
                    }
#pragma unroll
                    for (int r = 0; r < RS; ++r)
                        ui[r] = *reinterpret_cast<const T*>(b.own + (R0 + r) * RB);
                    load_rows(wi, xi);
                }
#pragma unroll
                for (int r = 0; r < RS; ++r)
                    step_epilogue<O, T, KIND, DMODE>(acc[r], ui[r], wi[r], xi[r], T{}, 0, wrow[r], wrow[r] + xdelta,
                                                     static_cast<T*>(nullptr), p.beta, coeff, c1, c2,
                                                     acc_d, comp_d);
#pragma unroll
                for (int r = 0; r < RS; ++r) wrow[r] += colstep;
                __syncwarp();
                if (lane0) {
                    mbar_arrive(&empty_z[zslot]);
                    if (c - 1 >= jlo) mbar_arrive(&empty_o[so_m]);
                }
                so_m = so_c;
                so_c = so_p;
                if (++so_p == no) so_p = 0;
                if (++zslot == nz) {
                    zslot = 0;
                    zpar ^= 1;
                }
            }
        };
        if constexpr (RS == G) {
            consume(std::integral_constant<int, 0>{});
        } else if constexpr (RS == 2) {
            if (grp == 0)
                consume(std::integral_constant<int, 0>{});
            else
                consume(std::integral_constant<int, 2>{});
        } else {
            if (grp == 0)
                consume(std::integral_constant<int, 0>{});
            else if (grp == 1)
                consume(std::integral_constant<int, 1>{});
            else if (grp == 2)
                consume(std::integral_constant<int, 2>{});
            else
                consume(std::integral_constant<int, 3>{});
        }
    }
    if constexpr (NDOT > 0) {
        __syncthreads();  // every staged column was consumed: the rings' shared memory is free
        const int uoff = p.u_off;
        double* outp = static_cast<double*>(p.dots_out);
        const int64_t dstride = p.dots_row_stride;
        grid_reduce<double, NDOT, true>(acc_d, NG * NCT / US, US, static_cast<double*>(p.partials),
                                        p.part_base + blockIdx.x, p.nparts, p.final_launch != 0, p.counter,
                                        [&](int d, int uu, double vv) { outp[d * dstride + uoff + uu] = vv; });
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline const void* ring_scaled_values(const Matrix& a, double s) {
    if (s == 1.0) return a.grp.vals.p;
    for (const auto& e : a.grp.scaled)
        if (e.first == s) return e.second->p;
    return nullptr;
}

// Launch the site-ring kernel for s if it applies; false = nothing launched.
template <int KIND, int DMODE = 0>
bool run_ring(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch) {
    const Matrix& a = *s.a;
    const GroupedMatrix& gm = a.grp;
    constexpr int NDOT = dots_of(DMODE);
    if (ctx.ring == 0 || ctx.kernel_variant != 1 || !gm.ok || !gm.ring_ok) return false;
    if (s.dots_mode != DMODE || units % 32 != 0) return false;
    // moment sums: whole-step launches only (a rank's interior / boundary launches keep the
    // kernels whose partial layout they share); CHEBFD_OPT_RING_DOTS = 0: never
    if (NDOT > 0 && (ctx.ring_dots == 0 || s.partial_base != 0 || !s.final_launch)) return false;
    const int64_t P = a.plane_rows, Ln = a.line_rows;
    const int64_t nrows = s.row1 - s.row0;
    if (P <= 0 || Ln <= 0 || nrows <= 0 || s.row0 % P != 0 || nrows % P != 0) return false;
    const int64_t lx = Ln / kGroupRows, ly = P / Ln, planes = nrows / P;
    if (ly % kRingSY != 0 || lx < 1 || lx > (1 << 24) || ly > (1 << 24)) return false;
    const void* svals = ring_scaled_values(a, s.alpha);
    if (!svals) return false;
    // 64-unit slabs (one CTA per SM) unless CHEBFD_OPT_SLAB_UNITS asks for 32 (two CTAs per SM).
    // Blocks of a multiple of 128 columns: 128-unit slabs on strips of two lines -- 2 KB instead
    // of 1 KB pieces of every row (ncu at n_b = 256: DRAM 63 % of its peak with 1 KB pieces
    // against 74 % with whole 1 KB rows at n_b = 64) and half the passes over the matrix:
    // C3 lattice n_b = 256 14.5 -> 13.5 ms per filter step, TI 512^2x4 n_b = 128 6.44 -> 6.15.
    // CHEBFD_OPT_SLAB_UNITS = 128 / 64 forces either.
    int us = (units % 64 == 0 && ctx.slab_units != 32) ? 64 : 32;
    if (units % 128 == 0 && (ctx.slab_units == 128 || (ctx.slab_units == 0 && units >= 128))) us = 128;
    const int SY = us == 128 ? 2 : kRingSY;
    // default (CHEBFD_OPT_RING = 1): lattices whose z-plane of the gathered block exceeds
    // twice the band budget (32 MB) -- measured with tools/ring_exp.py: C4 (1 GB planes) filter
    // 7.56 -> 6.36 ms per step, TI 512^2x8 n_b = 32 3.9 -> 3.45, TI 128^2x64 n_b = 64 (64 MB)
    // 4.5 -> 3.65, n_b = 256 (256 MB, four slabs) 15.5 -> 15.4; TI 64^3 n_b = 64 (16 MB planes,
    // L2-resident) 1.04 -> 1.15, where the SELL kernel stays.  2: wherever it applies
    // (planes of exactly 32 MB -- the C3 lattice at n_b = 32, the KPM block of its solve -- run
    // the ring kernel: filter 2.21 -> 1.97 ms per step, KPM of order 2000 2.95 -> 2.55 s)
    // x segment per CTA: 64 columns, halved down to 16 while the grid would be fewer than 24
    // waves of resident CTAs -- medium lattices (TI 64^3, 96^2 x 32) ran 1024 - 1536 long CTAs,
    // 3 - 10 waves with a ragged tail: TI 64^3 n_b = 64 1.00 -> 0.93 ms per filter step at 16
    // columns, n_b = 32 0.63 -> 0.50; 8 columns lose again to the apron columns
    const int64_t strips = ly / SY;
    const double slots = static_cast<double>(ctx.num_sms) * (us == 32 ? 2 : 1);
    auto waves = [&](int sx) { return static_cast<double>(strips * planes * ((lx + sx - 1) / sx)) / slots; };
    int segx_auto = 64;
    while (segx_auto > 16 && waves(segx_auto) < 24.0) segx_auto /= 2;
    // Below 32 MB planes (L2-resident): with the short segments and the last session's lighter
    // consumers the ring kernel also beats the SELL kernel from 8 MB planes on, given a dozen
    // waves of CTAs (TI 64^3 n_b = 32: filter 0.52 -> 0.50 ms per step, fused step 0.74 -> 0.79
    // of measured HBM; n_b = 64: 1.09 -> 0.93; TI 96^2 x 32 n_b = 32: 0.63 -> 0.70 of the
    // schedule's bytes); smaller lattices (48^3, 32^3) stay on the SELL kernel
    if (ctx.ring == 1) {
        const size_t plane_b = static_cast<size_t>(P) * units * 16;
        const size_t big = 2 * static_cast<size_t>(std::max<int64_t>(ctx.band_bytes, 0));
        if (plane_b < big && (plane_b * 4 < big || waves(ctx.ring_segx > 0 ? ctx.ring_segx : segx_auto) < 12.0))
            return false;
    }
    const size_t rb = static_cast<size_t>(us) * 16;
    const size_t os = (SY + 2) * kGroupRows * rb, zs = SY * kGroupRows * rb + SY * kRingMaxVals * 16;
    const int segx = static_cast<int>(std::min<int64_t>(lx, ctx.ring_segx > 0 ? ctx.ring_segx : segx_auto));
    const size_t plan_b = static_cast<size_t>(SY) * segx * 32;
    int no = us == 64 ? 5 : 5, nz = 3;
    if (ctx.ring_no > 0) no = std::min(ctx.ring_no, kRingMaxDepth);
    if (ctx.ring_nz > 0) nz = std::min(ctx.ring_nz, kRingMaxDepth);
    if (no < 4 || nz < 2) return false;
    const size_t smem = no * os + nz * zs + plan_b;
    if (smem > 220 * 1024) return false;
    // strips per band: the band's slice of the gathered operand within the band budget
    int64_t spb = 1;
    for (int64_t d = 1; d <= strips; ++d)
        if (strips % d == 0 && static_cast<size_t>(d * SY * Ln) * units * 16 <=
                                   static_cast<size_t>(std::max<int64_t>(ctx.band_bytes, 1)))
            spb = d;
    // CTA order 3 (default) = automatic: planes fastest where a wave of CTAs then still spans
    // eight or more strips (shallow slabs, C4: fused step 7.7 -> 7.4 ms), else bands of strips
    // with x segments fastest (the C3 lattice's 64 planes: 14.2 against 14.7 ms at n_b = 256)
    const int order = ctx.ring_order == 3 ? (planes * 8 <= ctx.num_sms ? 2 : 0) : ctx.ring_order;
    if (order == 2) {
        spb = strips;
    } else if (order != 0) {
        // a (segment, band) unit of CTAs about fills the GPU: all planes x spb strips
        spb = 1;
        for (int64_t d = 1; d <= strips; ++d)
            if (strips % d == 0 && d * planes <= std::max<int64_t>(ctx.ring_spb_ctas > 0 ? ctx.ring_spb_ctas : ctx.num_sms, planes))
                spb = d;
    }
    const int64_t nseg = (lx + segx - 1) / segx;
    const int64_t grid = strips * planes * nseg;
    if (grid >= (int64_t(1) << 31)) return false;
    if (NDOT > 0) {
        // the partial rows must fit the context's buffer as it is (graphs hold its address) and
        // the group tickets its 4 KB of counters
        if (!gm.ring_const_ok || ctx.ring_consts == 0 || grid > 32 * 1000) return false;
        if (static_cast<size_t>(reduce_rows_needed(grid)) * NDOT * us * sizeof(double) > ctx.partials.bytes) return false;
        ctx.counter.ensure(4096);
    }
    // rows per consumer thread: 2 by default (16 consumer warps per 64-unit strip CTA)
    int rs = ctx.ring_rows > 0 ? ctx.ring_rows : 2;
    if (rs != 4 && rs != 2 && rs != 1) rs = 2;
    if (us == 64 && rs == 1) rs = 2;  // 1024 consumer threads + the producer warp do not fit
    if (us == 128) rs = 2;
    // constant off-diagonal values (kernel parameters) where the matrix has them
    bool cv = gm.ring_const_ok && ctx.ring_consts != 0;
    RingConsts cc{};
    if (cv) {
        // the value a product uses: the real or the imaginary part, scaled as the grouped
        // value copies are (one IEEE multiply per component, group.cu scale_kernel)
        auto fill = [&](auto pat) {
            using P = decltype(pat);
            for (int k = 0; k < P::NC; ++k)
                for (int r = 0; r < kGroupRows; ++r) {
                    if (!((P::m(k) >> r) & 1u)) continue;
                    const int i = P::voff(k, r);
                    const double* v = gm.ring_consts[P::ID][i];
                    volatile double prod = ((P::im(k) >> r) & 1u) ? v[1] * s.alpha : v[0] * s.alpha;
                    cc.v[P::ID][i] = s.alpha == 1.0 ? (((P::im(k) >> r) & 1u) ? v[1] : v[0]) : prod;
                }
        };
        fill(PatTiMid{});
        fill(PatTiLo{});
        fill(PatTiHi{});
        // the row pairs' shared products (PatBase::pair_col) hold for these values?  Else the
        // kernels that read every value from memory
        bool share_ok = true;
        auto check = [&](auto pat) {
            using P = decltype(pat);
            if (!gm.ring_pat_present[P::ID]) return;  // no site runs this pattern
            for (int k = 0; k < P::NC; ++k) {
                if (!P::pair_col(k)) continue;
                const int ra = P::m(k) == 0x3u ? 0 : 2;
                const double va = cc.v[P::ID][P::voff(k, ra)], vb = cc.v[P::ID][P::voff(k, ra + 1)];
                if (va == 0.0 || !(vb == (P::pair_neg(k) ? -va : va))) share_ok = false;
            }
        };
        check(PatTiMid{});
        check(PatTiLo{});
        check(PatTiHi{});
        if (CFD_RING_SHARE != 0 && !share_ok) cv = false;
    }
    if (!cv) rs = 2;
    if (us == 32 && rs == 4) rs = 2;
    if (NDOT > 0 && (!cv || rs != 2)) return false;
    void (*kernel)(const StepParams, const RingParams, const RingConsts, const RingMaps) =
        us == 128 ? (cv ? step_ring_kernel<KIND, 128, 2, true, 2> : step_ring_kernel<KIND, 128, 2, false, 2>)
        : !cv ? (us == 64 ? step_ring_kernel<KIND, 64, 2, false> : step_ring_kernel<KIND, 32, 2, false>)
        : us == 64 ? (rs == 4 ? step_ring_kernel<KIND, 64, 4, true> : step_ring_kernel<KIND, 64, 2, true>)
                   : (rs == 2 ? step_ring_kernel<KIND, 32, 2, true> : step_ring_kernel<KIND, 32, 1, true>);
    if constexpr (NDOT > 0)
        kernel = us == 128  ? step_ring_kernel<KIND, 128, 2, true, 2, DMODE>
                 : us == 64 ? step_ring_kernel<KIND, 64, 2, true, kRingSY, DMODE>
                            : step_ring_kernel<KIND, 32, 2, true, kRingSY, DMODE>;
    static thread_local std::map<std::pair<const void*, int>, size_t> attr_set;
    auto& cur = attr_set[std::make_pair(reinterpret_cast<const void*>(kernel), ctx.device)];
    if (cur < smem) {
        CFD_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        cur = smem;
    }
    for (int u0 = 0; u0 < units; u0 += us) {
        StepParams p{};
        p.row0 = s.row0;
        p.row1 = s.row1;
        p.halo_lo = a.part.halo_lo;
        p.pitch = pitch;
        p.u_off = u0;
        p.US = us;
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
        p.dots_row_stride = units;
        p.partials = ctx.partials.p;
        p.part_base = 0;
        p.nparts = static_cast<int>(grid);
        p.final_launch = 1;
        p.counter = ctx.counter.as<unsigned>();
        RingParams rp{};
        rp.plan = gm.ring_plan.as<int4>();
        rp.cols = gm.cols.as<int>();
        rp.vals = svals;
        rp.lx = static_cast<int>(lx);
        rp.ly = static_cast<int>(ly);
        rp.planes = static_cast<int>(planes);
        rp.segx = segx;
        rp.nseg = static_cast<int>(nseg);
        rp.spb = static_cast<int>(spb);
        rp.nbands = static_cast<int>(strips / spb);
        rp.order = order;
        rp.no = no;
        rp.nz = nz;
        rp.full = (us == units && pitch == units) ? 1 : 0;
        // tensor-map copies: CHEBFD_OPT_RING_TMAP 1 (default) wherever a slab is narrower
        // than the row, 2 always, 0 never (per-row 1D copies for slabs)
        RingMaps maps{};
        rp.tmap = 0;
        if ((ctx.ring_tmap == 2 || (ctx.ring_tmap == 1 && !rp.full)) &&
            make_ring_maps(maps, s.in, a.part.ext_rows(), pitch, us))
            rp.tmap = 1;
        const bool pdl = s.pdl_ok && ctx.pdl == 2;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(grid));
        cfg.blockDim = dim3(static_cast<unsigned>((kGroupRows / rs) * SY * us + 64));
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CFD_CUDA(cudaLaunchKernelEx(&cfg, kernel, p, rp, cc, maps));
        CFD_CUDA(cudaGetLastError());
        ctx.launches++;
        ctx.ring_launches++;
        ctx.band_launches++;
    }
    if (s.grid_used) *s.grid_used = static_cast<int>(grid);
    return true;
}

inline bool dispatch_ring(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch) {
    if (s.dots_mode != 0) {
        if (s.kind_step != kStepRecur) return false;
        if (s.dots_mode == 4) return run_ring<kStepRecur, 4>(ctx, s, st, units, pitch);
        if (s.dots_mode == 5) return run_ring<kStepRecur, 5>(ctx, s, st, units, pitch);
        if (s.dots_mode == 6) return run_ring<kStepRecur, 6>(ctx, s, st, units, pitch);
        return false;
    }
    switch (s.kind_step) {
        case kStepFused: return run_ring<kStepFused>(ctx, s, st, units, pitch);
        case kStepRecur: return run_ring<kStepRecur>(ctx, s, st, units, pitch);
        case kStepFusedX2: return run_ring<kStepFusedX2>(ctx, s, st, units, pitch);
        case kStepFusedX3: return run_ring<kStepFusedX3>(ctx, s, st, units, pitch);
    }
    return false;
}

}  // namespace
}  // namespace cfd
