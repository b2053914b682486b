// Grouped form of the matrix (internal.hpp GroupedMatrix): rows 4g .. 4g+3 share one merged
// list of gathered columns.  Built on the device from the CSR the SELL build reads.
//
// The merge keeps every row's own entry order -- the reference accumulates a row's sum in
// CSR order (kernels.hpp:56-60), and so must we to match it bit for bit.  All rows of a CSR
// are subsequences of one total order (the global column order), but the builder only sees
// extended-row indices, whose order differs from it on ring-wrapped halos.  So the merge is
// order-free: a head column is "safe" when no other row still holds it behind its head;
// the safe head with the smallest index is emitted for every row whose head it is.  The
// smallest remaining column in the rows' common order is always safe, so rows of a
// consistently ordered CSR always merge into their exact union.  If no head is safe (rows
// in inconsistent orders), one row's head is emitted unshared, which is always valid.
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include "internal.hpp"
#include "group_patterns.hpp"

namespace cfd {
namespace {

constexpr unsigned kColBits = 28;
constexpr unsigned kColMask = (1u << kColBits) - 1u;

struct GroupRows {
    int col[kGroupRows][kGroupMaxRowLen];
    int len[kGroupRows];
    int64_t off[kGroupRows];  // CSR offset of each row's first entry
};

// load the mapped columns of group g's rows; false if a row is too long / a column does not fit
__device__ bool load_group(const int64_t* __restrict__ offs, const int64_t* __restrict__ gcols,
                           int64_t rows, int64_t g, const ColMap& cm, GroupRows& gr, int* err) {
    bool ok = true;
    for (int r = 0; r < kGroupRows; ++r) {
        const int64_t row = g * kGroupRows + r;
        gr.len[r] = 0;
        gr.off[r] = 0;
        if (row >= rows) continue;
        const int64_t b = offs[row], e = offs[row + 1];
        gr.off[r] = b;
        if (e - b > kGroupMaxRowLen) {
            ok = false;
            continue;
        }
        gr.len[r] = static_cast<int>(e - b);
        for (int j = 0; j < gr.len[r]; ++j) {
            const int64_t c = cm.map(gcols[b + j]);
            if (c < 0) atomicExch(err, 1);
            if (c < 0 || c > static_cast<int64_t>(kColMask)) ok = false;
            gr.col[r][j] = static_cast<int>(c);
        }
    }
    return ok;
}

// One merge step: the column to emit and the rows that take it (mask); advances the heads.
__device__ __forceinline__ bool merge_next(const GroupRows& gr, int (&head)[kGroupRows], int& col,
                                           unsigned& mask) {
    int best = -1;
    bool any = false;
    for (int r = 0; r < kGroupRows; ++r) {
        if (head[r] >= gr.len[r]) continue;
        any = true;
        const int x = gr.col[r][head[r]];
        if (best >= 0 && x >= best) continue;
        bool safe = true;
        for (int s = 0; s < kGroupRows && safe; ++s) {
            if (s == r || head[s] >= gr.len[s] || gr.col[s][head[s]] == x) continue;
            for (int j = head[s] + 1; j < gr.len[s]; ++j)
                if (gr.col[s][j] == x) {
                    safe = false;
                    break;
                }
        }
        if (safe) best = x;
    }
    if (!any) return false;
    mask = 0u;
    if (best >= 0) {
        col = best;
        for (int r = 0; r < kGroupRows; ++r)
            if (head[r] < gr.len[r] && gr.col[r][head[r]] == best) {
                mask |= 1u << r;
                ++head[r];
            }
    } else {  // inconsistent row orders: the first pending row's head, unshared
        for (int r = 0; r < kGroupRows; ++r)
            if (head[r] < gr.len[r]) {
                col = gr.col[r][head[r]];
                mask = 1u << r;
                ++head[r];
                break;
            }
    }
    return true;
}

// pass 1: per group, padded column count and value count
__global__ void group_count_kernel(const int64_t* __restrict__ offs, const int64_t* __restrict__ gcols,
                                   int64_t rows, int64_t ngroups, ColMap cm, int* __restrict__ cnt_c,
                                   int* __restrict__ cnt_v, int* __restrict__ flags) {
    const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (g >= ngroups) return;
    GroupRows gr;
    if (!load_group(offs, gcols, rows, g, cm, gr, flags + 1)) {
        atomicExch(flags, 1);
        cnt_c[g] = cnt_v[g] = 0;
        return;
    }
    int head[kGroupRows] = {0, 0, 0, 0};
    int col = 0, n = 0, nv = 0;
    unsigned mask = 0;
    while (merge_next(gr, head, col, mask)) {
        ++n;
        nv += __popc(mask);
    }
    cnt_c[g] = (n + 3) & ~3;
    cnt_v[g] = nv;
}

// pass 2: per tile, segment sizes (ints incl. the header; values, even) and their maxima
__global__ void tile_size_kernel(const int* __restrict__ cnt_c, const int* __restrict__ cnt_v,
                                 int64_t ngroups, int64_t ntiles, int64_t* __restrict__ tc,
                                 int64_t* __restrict__ tv, int* __restrict__ maxima, TileMap tm) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t > ntiles) return;
    if (t == ntiles) {  // scan sentinel
        tc[t] = tv[t] = 0;
        return;
    }
    int c = 4 * kTileGroups, v = 0;
    for (int i = 0; i < kTileGroups; ++i) {
        const int64_t g = tm.first_row(t, i) / kGroupRows;
        if (g < ngroups) {
            c += cnt_c[g];
            v += cnt_v[g];
        }
    }
    v = (v + 1) & ~1;
    tc[t] = c;
    tv[t] = v;
    atomicMax(&maxima[0], c);
    atomicMax(&maxima[1], v);
}

// does the merged group (n columns, their masks and indices) equal library pattern P, with
// the group's own rows own0 .. own0 + 3 where P expects them?
template <class P>
__device__ bool matches(const unsigned char* masks, const int* cols, int n, int64_t own0,
                        const double2* vseg) {
    if (n != P::NC) return false;
    for (int k = 0; k < P::NC; ++k)
        if (masks[k] != P::m(k)) return false;
    for (int r = 0; r < kGroupRows; ++r)
        if (cols[P::OWN + r] != own0 + r) return false;
    // the entries the pattern multiplies as purely real / imaginary must be so
    for (int k = 0; k < P::NC; ++k)
        for (int r = 0; r < kGroupRows; ++r) {
            if (!((P::m(k) >> r) & 1u)) continue;
            const double2 v = vseg[P::voff(k, r)];
            if (((P::re(k) >> r) & 1u) && v.y != 0.0) return false;
            if (((P::im(k) >> r) & 1u) && v.x != 0.0) return false;
        }
    return true;
}

// pass 3: headers (with the static pattern id, 0 = none), packed columns and values
template <class M>
__global__ void group_fill_kernel(const int64_t* __restrict__ offs, const int64_t* __restrict__ gcols,
                                  const M* __restrict__ gvals, int64_t rows, int64_t ngroups,
                                  ColMap cm, const int* __restrict__ cnt_c,
                                  const int* __restrict__ cnt_v, const int64_t* __restrict__ tile_cptr,
                                  const int64_t* __restrict__ tile_vptr, int* __restrict__ cols,
                                  M* __restrict__ vals, int64_t halo_lo, int cplx, TileMap tm) {
    // one thread per (tile, group slot)
    const int64_t slot = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t ntg = (ngroups + kTileGroups - 1) / kTileGroups * kTileGroups;
    if (slot >= ntg) return;
    const int64_t t = slot / kTileGroups;
    const int gi = static_cast<int>(slot % kTileGroups);
    const int64_t g = tm.first_row(t, gi) / kGroupRows;
    int coff = 4 * kTileGroups, voff = 0;
    for (int i = 0; i < gi; ++i) {
        const int64_t q = tm.first_row(t, i) / kGroupRows;
        if (q < ngroups) {
            coff += cnt_c[q];
            voff += cnt_v[q];
        }
    }
    int* seg = cols + tile_cptr[t];
    M* vseg = vals + tile_vptr[t];
    int4* hdr = reinterpret_cast<int4*>(seg) + gi;
    if (g >= ngroups) {
        *hdr = make_int4(coff, voff, 0, 0);
        return;
    }
    GroupRows gr;
    int dummy = 0;
    load_group(offs, gcols, rows, g, cm, gr, &dummy);
    int head[kGroupRows] = {0, 0, 0, 0};
    int col = 0, n = 0, nv = 0;
    unsigned mask = 0;
    int last = 0;
    unsigned char masks[32];
    int ucols[32];
    while (merge_next(gr, head, col, mask)) {
        seg[coff + n] = static_cast<int>(static_cast<unsigned>(col) | (mask << kColBits));
        last = col;
        if (n < 32) {
            masks[n] = static_cast<unsigned char>(mask);
            ucols[n] = col;
        }
        ++n;
        for (int r = 0; r < kGroupRows; ++r)
            if (mask & (1u << r)) vseg[voff + nv++] = gvals[gr.off[r] + head[r] - 1];
    }
    const int npad = (n + 3) & ~3;
    for (int k = n; k < npad; ++k) seg[coff + k] = last;  // mask 0: gathered, never used
    int pat = 0;
    if constexpr (sizeof(M) == 16) {
        if (cplx && n <= 32 && g * kGroupRows + kGroupRows <= rows) {
            const int64_t own0 = g * kGroupRows + halo_lo;
            const double2* gv = reinterpret_cast<const double2*>(vseg + voff);
            if (matches<PatTiMid>(masks, ucols, n, own0, gv)) pat = 1;
            else if (matches<PatTiLo>(masks, ucols, n, own0, gv)) pat = 2;
            else if (matches<PatTiHi>(masks, ucols, n, own0, gv)) pat = 3;
        }
    }
    *hdr = make_int4(coff, voff, npad, pat);
    // the tile's last slot zero-fills the padding value of an odd count (linear tiles: the
    // last group of the matrix may sit before unused slots)
    if (gi == kTileGroups - 1 || (tm.line_rows == 0 && g == ngroups - 1)) {
        const int64_t vend = tile_vptr[t + 1] - tile_vptr[t];
        for (int64_t k = voff + nv; k < vend; ++k) vseg[k] = M{};
    }
}

__global__ void scale_kernel(double* __restrict__ out, const double* __restrict__ in, int64_t n,
                             double s) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = __dmul_rn(in[i], s);
}


// ---- site-ring plan (step_ring.cuh) ---------------------------------------------------
// static site of pattern P: its x -+ 1 / y -+ 1 column blocks are the lattice neighbours' rows
template <class P>
__device__ bool ring_neighbours_ok(const int* c, int64_t own0, int64_t line_rows) {
    for (int r = 0; r < kGroupRows; ++r) {
        if (static_cast<int64_t>(c[P::OWN - 8 + r] & kColMask) != own0 - line_rows + r) return false;
        if (static_cast<int64_t>(c[P::OWN - 4 + r] & kColMask) != own0 - kGroupRows + r) return false;
        if (static_cast<int64_t>(c[P::OWN + 4 + r] & kColMask) != own0 + kGroupRows + r) return false;
        if (static_cast<int64_t>(c[P::OWN + 8 + r] & kColMask) != own0 + line_rows + r) return false;
    }
    return true;
}

__global__ void ring_plan_kernel(const int64_t* __restrict__ tile_cptr,
                                 const int64_t* __restrict__ tile_vptr, const int* __restrict__ cols,
                                 int64_t ngroups, int64_t halo_lo, int64_t line_rows,
                                 int4* __restrict__ plan, int* __restrict__ bad) {
    const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (g >= ngroups) return;
    const int64_t t = g / kTileGroups;
    const int gi = static_cast<int>(g % kTileGroups);
    const int* seg = cols + tile_cptr[t];
    const int4 h = reinterpret_cast<const int4*>(seg)[gi];
    const int* c = seg + h.x;
    int nv = 0;
    for (int k = 0; k < h.z; ++k) nv += __popc(static_cast<unsigned>(c[k]) >> kColBits);
    if (nv > kRingMaxVals) atomicExch(bad, 1);
    const int64_t voff = tile_vptr[t] + h.y;
    const int64_t own0 = g * kGroupRows + halo_lo;
    int4 a;
    bool ok = true;
    if (h.w == 1) {
        a = make_int4(c[0] & kColMask, c[1] & kColMask, c[22] & kColMask, c[23] & kColMask);
        ok = ring_neighbours_ok<PatTiMid>(c, own0, line_rows);
    } else if (h.w == 2) {
        a = make_int4(-1, -1, c[20] & kColMask, c[21] & kColMask);
        ok = ring_neighbours_ok<PatTiLo>(c, own0, line_rows);
    } else if (h.w == 3) {
        a = make_int4(c[0] & kColMask, c[1] & kColMask, -1, -1);
        ok = ring_neighbours_ok<PatTiHi>(c, own0, line_rows);
    } else {
        const int64_t coff = tile_cptr[t] + h.x;
        a = make_int4(static_cast<int>(coff & 0xFFFFFFFFll), static_cast<int>(coff >> 32), h.z, 0);
    }
    if (!ok) atomicExch(bad, 1);
    plan[2 * g] = a;
    plan[2 * g + 1] =
        make_int4(static_cast<int>(voff & 0xFFFFFFFFll), static_cast<int>(voff >> 32), h.w, nv);
}


// first static group of each pattern (reference values for the constant check)
__global__ void ring_first_kernel(const int4* __restrict__ plan, int64_t ngroups,
                                  unsigned long long* __restrict__ first) {
    const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (g >= ngroups) return;
    const int pat = plan[2 * g + 1].z;
    if (pat >= 1 && pat <= 3) atomicMin(&first[pat - 1], static_cast<unsigned long long>(g));
}

// do all static groups of a pattern hold the reference group's values, the own-row diagonal
// entries (k = OWN + r, row r) aside?
template <class P>
__device__ bool ring_same_values(const double2* v, const double2* ref) {
    for (int k = 0; k < P::NC; ++k)
        for (int r = 0; r < kGroupRows; ++r) {
            if (!((P::m(k) >> r) & 1u) || k == P::OWN + r) continue;
            const int i = P::voff(k, r);
            if (__double_as_longlong(v[i].x) != __double_as_longlong(ref[i].x) ||
                __double_as_longlong(v[i].y) != __double_as_longlong(ref[i].y))
                return false;
        }
    return true;
}

__global__ void ring_const_kernel(const int4* __restrict__ plan, const double2* __restrict__ vals,
                                  int64_t ngroups, const unsigned long long* __restrict__ first,
                                  int* __restrict__ bad) {
    const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (g >= ngroups) return;
    const int4 b = plan[2 * g + 1];
    if (b.z < 1 || b.z > 3) return;
    const int4 rb = plan[2 * first[b.z - 1] + 1];
    auto off = [](const int4& q) {
        return static_cast<int64_t>(static_cast<unsigned>(q.x)) | (static_cast<int64_t>(q.y) << 32);
    };
    const double2* v = vals + off(b);
    const double2* ref = vals + off(rb);
    bool ok;
    if (b.z == 1)
        ok = ring_same_values<PatTiMid>(v, ref);
    else if (b.z == 2)
        ok = ring_same_values<PatTiLo>(v, ref);
    else
        ok = ring_same_values<PatTiHi>(v, ref);
    if (!ok) atomicExch(bad, 1);
}

}  // namespace

// plan of the site-ring step kernel: complex lattice operators whose rows are whole sites in
// linear tiles; leaves gm.ring_ok = false where it does not apply
static void build_ring_plan(Matrix& m, cudaStream_t st) {
    GroupedMatrix& gm = m.grp;
    gm.ring_ok = false;
    const int64_t rows = m.part.local;
    if (!gm.ok || !m.kind || m.line_rows <= 0 || m.plane_rows <= 0 || gm.il_line_rows != 0 ||
        m.line_rows % kGroupRows != 0 || m.plane_rows % m.line_rows != 0 || rows % m.plane_rows != 0)
        return;
    const int64_t ngroups = rows / kGroupRows;
    gm.ring_plan.ensure(sizeof(int4) * 2 * ngroups);
    DeviceBuffer bad(sizeof(int));
    CFD_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    ring_plan_kernel<<<static_cast<unsigned>((ngroups + 127) / 128), 128, 0, st>>>(
        gm.tile_cptr.as<int64_t>(), gm.tile_vptr.as<int64_t>(), gm.cols.as<int>(), ngroups,
        m.part.halo_lo, m.line_rows, gm.ring_plan.as<int4>(), bad.as<int>());
    CFD_CUDA(cudaGetLastError());
    int h = 0;
    CFD_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CFD_CUDA(cudaStreamSynchronize(st));
    gm.ring_ok = h == 0;
    gm.ring_const_ok = false;
    if (!gm.ring_ok) return;
    // constant off-diagonal values per pattern?
    DeviceBuffer first(3 * sizeof(unsigned long long));
    CFD_CUDA(cudaMemsetAsync(first.p, 0xFF, 3 * sizeof(unsigned long long), st));
    CFD_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    const unsigned grid = static_cast<unsigned>((ngroups + 127) / 128);
    ring_first_kernel<<<grid, 128, 0, st>>>(gm.ring_plan.as<int4>(), ngroups,
                                            first.as<unsigned long long>());
    ring_const_kernel<<<grid, 128, 0, st>>>(gm.ring_plan.as<int4>(), gm.vals.as<double2>(), ngroups,
                                            first.as<unsigned long long>(), bad.as<int>());
    CFD_CUDA(cudaGetLastError());
    unsigned long long hf[3];
    CFD_CUDA(cudaMemcpyAsync(hf, first.p, sizeof(hf), cudaMemcpyDeviceToHost, st));
    CFD_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CFD_CUDA(cudaStreamSynchronize(st));
    if (h != 0) return;
    for (int q = 0; q < 3; ++q) {
        gm.ring_pat_present[q] = hf[q] != ~0ull;
        if (hf[q] == ~0ull) continue;  // pattern absent: its constants are never used
        int4 pb;
        CFD_CUDA(cudaMemcpy(&pb, gm.ring_plan.as<int4>() + 2 * hf[q] + 1, sizeof(int4),
                            cudaMemcpyDeviceToHost));
        const int64_t voff = static_cast<int64_t>(static_cast<unsigned>(pb.x)) |
                             (static_cast<int64_t>(pb.y) << 32);
        const int nv = std::min(pb.w, kRingMaxVals);
        CFD_CUDA(cudaMemcpy(gm.ring_consts[q], gm.vals.as<double2>() + voff,
                            sizeof(double) * 2 * nv, cudaMemcpyDeviceToHost));
    }
    gm.ring_const_ok = true;
}

void build_grouped(Context& ctx, Matrix& m, const int64_t* d_offs, const int64_t* d_cols,
                   const void* d_vals, cudaStream_t st) {
    GroupedMatrix& gm = m.grp;
    gm.ok = false;
    gm.scaled.clear();
    const int64_t rows = m.part.local;
    if (rows <= 0 || m.max_row_len > kGroupMaxRowLen ||
        m.part.ext_rows() > static_cast<int64_t>(kColMask))
        return;
    const int64_t ngroups = (rows + kGroupRows - 1) / kGroupRows;
    const int64_t ntiles = (ngroups + kTileGroups - 1) / kTileGroups;
    const ColMap cm = m.part.compact ? ColMap{0, m.part.ext_rows(), 0, 0, 0, 0} : colmap_of(m.part);
    // lattice operators: tiles of L lines x 16 / L sites where the lines divide evenly
    gm.il_line_rows = 0;
    gm.il_lines = 1;
    const int L = ctx.group_lines;
    if ((L == 2 || L == 4) && m.line_rows > 0 && m.line_rows % (kGroupRows * (kTileGroups / L)) == 0 &&
        rows % (L * m.line_rows) == 0) {
        gm.il_line_rows = m.line_rows;
        gm.il_lines = L;
    }
    const TileMap tm = tilemap_of(gm);
    DeviceBuffer cnt_c(sizeof(int) * ngroups), cnt_v(sizeof(int) * ngroups);
    DeviceBuffer tc(sizeof(int64_t) * (ntiles + 1)), tv(sizeof(int64_t) * (ntiles + 1));
    DeviceBuffer flags(sizeof(int) * 4);  // unsupported, column error, max tile ints, max tile values
    CFD_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int) * 4, st));
    // the compact map is an identity over extended rows: halo_lo must still offset own rows
    ColMap cmf = cm;
    group_count_kernel<<<static_cast<unsigned>((ngroups + 127) / 128), 128, 0, st>>>(
        d_offs, d_cols, rows, ngroups, cmf, cnt_c.as<int>(), cnt_v.as<int>(), flags.as<int>());
    CFD_CUDA(cudaGetLastError());
    tile_size_kernel<<<static_cast<unsigned>((ntiles + 1 + 127) / 128), 128, 0, st>>>(
        cnt_c.as<int>(), cnt_v.as<int>(), ngroups, ntiles, tc.as<int64_t>(), tv.as<int64_t>(),
        flags.as<int>() + 2, tm);
    CFD_CUDA(cudaGetLastError());
    gm.tile_cptr.ensure(sizeof(int64_t) * (ntiles + 1));
    gm.tile_vptr.ensure(sizeof(int64_t) * (ntiles + 1));
    size_t tmp_bytes = 0;
    CFD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, tc.as<int64_t>(),
                                           gm.tile_cptr.as<int64_t>(), ntiles + 1, st));
    DeviceBuffer tmp(std::max<size_t>(tmp_bytes, 16));
    CFD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, tc.as<int64_t>(),
                                           gm.tile_cptr.as<int64_t>(), ntiles + 1, st));
    CFD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, tv.as<int64_t>(),
                                           gm.tile_vptr.as<int64_t>(), ntiles + 1, st));
    int h[4] = {0, 0, 0, 0};
    int64_t ncols = 0, nvals = 0;
    CFD_CUDA(cudaMemcpyAsync(h, flags.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    CFD_CUDA(cudaMemcpyAsync(&ncols, gm.tile_cptr.as<int64_t>() + ntiles, sizeof(int64_t),
                             cudaMemcpyDeviceToHost, st));
    CFD_CUDA(cudaMemcpyAsync(&nvals, gm.tile_vptr.as<int64_t>() + ntiles, sizeof(int64_t),
                             cudaMemcpyDeviceToHost, st));
    CFD_CUDA(cudaStreamSynchronize(st));
    if (h[0] || h[1]) return;  // unsupported shape (the SELL build reports column errors)
    gm.ntiles = ntiles;
    gm.ncols = ncols;
    gm.nvals = nvals;
    gm.max_tile_cols = h[2];
    gm.max_tile_vals = h[3];
    gm.cols.ensure(sizeof(int) * std::max<int64_t>(ncols, 4));
    gm.vals.ensure((m.kind ? 16 : 8) * std::max<int64_t>(nvals, 2));
    const int64_t ntg = ntiles * kTileGroups;
    const unsigned grid = static_cast<unsigned>((ntg + 127) / 128);
    if (m.kind)
        group_fill_kernel<double2><<<grid, 128, 0, st>>>(
            d_offs, d_cols, static_cast<const double2*>(d_vals), rows, ngroups, cmf, cnt_c.as<int>(),
            cnt_v.as<int>(), gm.tile_cptr.as<int64_t>(), gm.tile_vptr.as<int64_t>(),
            gm.cols.as<int>(), gm.vals.as<double2>(), m.part.halo_lo, 1, tm);
    else
        group_fill_kernel<double><<<grid, 128, 0, st>>>(
            d_offs, d_cols, static_cast<const double*>(d_vals), rows, ngroups, cmf, cnt_c.as<int>(),
            cnt_v.as<int>(), gm.tile_cptr.as<int64_t>(), gm.tile_vptr.as<int64_t>(),
            gm.cols.as<int>(), gm.vals.as<double>(), m.part.halo_lo, 0, tm);
    CFD_CUDA(cudaGetLastError());
    CFD_CUDA(cudaStreamSynchronize(st));
    gm.ok = true;
    build_ring_plan(m, st);
}

// values of the grouped form pre-multiplied by s (kept beside Matrix::scaled, same keys)
void ensure_scaled_grouped(Context& ctx, Matrix& a, double s, cudaStream_t st) {
    GroupedMatrix& gm = a.grp;
    if (!gm.ok) return;
    for (const auto& e : gm.scaled)
        if (e.first == s) return;
    if (gm.scaled.size() >= 4) gm.scaled.erase(gm.scaled.begin());
    const int64_t n = std::max<int64_t>(gm.nvals, 2) * (a.kind ? 2 : 1);
    auto buf = std::make_unique<DeviceBuffer>(sizeof(double) * n);
    const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, ctx.num_sms * 8));
    scale_kernel<<<grid, 256, 0, st>>>(buf->as<double>(), gm.vals.as<double>(), n, s);
    CFD_CUDA(cudaGetLastError());
    gm.scaled.emplace_back(s, std::move(buf));
}

}  // namespace cfd
