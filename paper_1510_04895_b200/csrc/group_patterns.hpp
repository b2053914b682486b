// Static group patterns shared by the grouped-matrix builder (group.cu) and the row-group
// step kernel (step_group.cuh).
#pragma once
#include "internal.hpp"

namespace cfd {
namespace {

// ---- static group patterns -----------------------------------------------------------------
// A pattern is the row-mask sequence of a group's merged columns plus the position of the
// group's own four rows among them.  Groups whose sequence equals a library pattern (the
// builder compares, group.cu) run straight-line code: every gather issued up front, every
// value at a fixed shared-memory offset, no per-column tests.  Library: the sites of the
// topological-insulator stencil (models.cpp:80-139) away from the x / y wrap -- blocks
// z-1 | y-1 | x-1 | site | x+1 | y+1 | z+1 in column order -- in the slab's bottom plane,
// its interior and its top plane.  Everything else takes the generic path.
//
// A pattern also states which entries are purely real or purely imaginary (the builder
// checks the stored values).  For a = (a, 0): a u = (a u_r - 0 u_i, a u_i + 0 u_r) rounds to
// (a u_r, a u_i) exactly, since x -+ 0 = x for x != 0; likewise a = (0, b) gives
// (-(b u_i), b u_r).  The results equal the reference's four-multiply product bit for bit
// for finite inputs, except the sign of an exact zero when a product itself is zero.
template <class D>
struct PatBase {
    // values before column k's row r in the group's value stream
    __host__ __device__ static constexpr int voff(int k, int r) {
        int n = 0;
        for (int j = 0; j < k; ++j)
            for (int q = 0; q < kGroupRows; ++q) n += (D::m(j) >> q) & 1;
        for (int q = 0; q < r; ++q) n += (D::m(k) >> q) & 1;
        return n;
    }
    // x / y neighbour columns (positions 0..7 and 12..19 after the z-1 columns) are read by
    // the two rows of one row pair (mask 0x3 or 0xC), with values of equal magnitude: every
    // nonzero entry of hop[j] = -t (G1 - i G^{j+1}) / 2 is +-t/2 or +-i t/2 (models.cpp:88-93).
    // pair_neg(k): the upper row's real / imaginary part has the opposite sign to the lower
    // row's, so both rows' products are +-(v g_r), +-(v g_i) of ONE value v: two multiplies per
    // column instead of four ((-v) g = -(v g) and a + (-p) = a - p exactly).  The launcher
    // checks the relation on the actual values (step_ring.cuh run_ring).
    __host__ __device__ static constexpr bool pair_col(int k) {
        const int q = k - (D::OWN - 8);
        return ((q >= 0 && q < 8) || (q >= 12 && q < 20)) && (D::m(k) == 0x3u || D::m(k) == 0xCu);
    }
    __host__ __device__ static constexpr bool pair_neg(int k) {
        return (0x930C6u >> (k - (D::OWN - 8))) & 1u;
    }
};
struct PatTiMid : PatBase<PatTiMid> {
    static constexpr int NC = 24, OWN = 10, ID = 0;
    __host__ __device__ static constexpr unsigned m(int k) {
        constexpr unsigned char t[NC] = {0x4, 0x2, 0xC, 0xC, 0x3, 0x3, 0xC, 0xC, 0x3, 0x3, 0x5, 0xA,
                                         0x5, 0xA, 0xC, 0xC, 0x3, 0x3, 0xC, 0xC, 0x3, 0x3, 0x8, 0x1};
        return t[k];
    }
    // rows whose value at column k is purely real / purely imaginary (the hopping and
    // on-site terms of models.cpp:88-139 are): their products need two multiplies, not four
    __host__ __device__ static constexpr unsigned re(int k) {
        constexpr unsigned char t[NC] = {0x4, 0x2, 0x4, 0x8, 0x1, 0x2, 0xC, 0xC, 0x3, 0x3, 0x5, 0xA, 0x5, 0xA, 0xC, 0xC, 0x3, 0x3, 0x4, 0x8, 0x1, 0x2, 0x8, 0x1};
        return t[k];
    }
    __host__ __device__ static constexpr unsigned im(int k) {
        constexpr unsigned char t[NC] = {0x0, 0x0, 0x8, 0x4, 0x2, 0x1, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x8, 0x4, 0x2, 0x1, 0x0, 0x0};
        return t[k];
    }
};
struct PatTiLo : PatBase<PatTiLo> {  // no z-1 neighbours
    static constexpr int NC = 22, OWN = 8, ID = 1;
    __host__ __device__ static constexpr unsigned m(int k) {
        constexpr unsigned char t[NC] = {0xC, 0xC, 0x3, 0x3, 0xC, 0xC, 0x3, 0x3, 0x5, 0xA, 0x5,
                                         0xA, 0xC, 0xC, 0x3, 0x3, 0xC, 0xC, 0x3, 0x3, 0x8, 0x1};
        return t[k];
    }
    // rows whose value at column k is purely real / purely imaginary (the hopping and
    // on-site terms of models.cpp:88-139 are): their products need two multiplies, not four
    __host__ __device__ static constexpr unsigned re(int k) {
        constexpr unsigned char t[NC] = {0x4, 0x8, 0x1, 0x2, 0xC, 0xC, 0x3, 0x3, 0x5, 0xA, 0x5, 0xA, 0xC, 0xC, 0x3, 0x3, 0x4, 0x8, 0x1, 0x2, 0x8, 0x1};
        return t[k];
    }
    __host__ __device__ static constexpr unsigned im(int k) {
        constexpr unsigned char t[NC] = {0x8, 0x4, 0x2, 0x1, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x8, 0x4, 0x2, 0x1, 0x0, 0x0};
        return t[k];
    }
};
struct PatTiHi : PatBase<PatTiHi> {  // no z+1 neighbours
    static constexpr int NC = 22, OWN = 10, ID = 2;
    __host__ __device__ static constexpr unsigned m(int k) {
        constexpr unsigned char t[NC] = {0x4, 0x2, 0xC, 0xC, 0x3, 0x3, 0xC, 0xC, 0x3, 0x3, 0x5,
                                         0xA, 0x5, 0xA, 0xC, 0xC, 0x3, 0x3, 0xC, 0xC, 0x3, 0x3};
        return t[k];
    }
    // rows whose value at column k is purely real / purely imaginary (the hopping and
    // on-site terms of models.cpp:88-139 are): their products need two multiplies, not four
    __host__ __device__ static constexpr unsigned re(int k) {
        constexpr unsigned char t[NC] = {0x4, 0x2, 0x4, 0x8, 0x1, 0x2, 0xC, 0xC, 0x3, 0x3, 0x5, 0xA, 0x5, 0xA, 0xC, 0xC, 0x3, 0x3, 0x4, 0x8, 0x1, 0x2};
        return t[k];
    }
    __host__ __device__ static constexpr unsigned im(int k) {
        constexpr unsigned char t[NC] = {0x0, 0x0, 0x8, 0x4, 0x2, 0x1, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x0, 0x8, 0x4, 0x2, 0x1};
        return t[k];
    }
};

}  // namespace
}  // namespace cfd
