// Row partitioning and halo planning for the distributed filter (host only).
//
// The reference is single-address-space; the paper's GHOST
// distribution (MPI row partition + halo exchange) is
// restated here for one process per B200: contiguous row ranges on lattice
// planes, halos = the contiguous runs of neighbour rows the local rows read.
#include <algorithm>
#include <cstring>
#include <vector>

#include "capi_common.hpp"

namespace cfd {

Partition plan_rows(const HostCsr& csr, int64_t r0, int64_t r1, const std::vector<int64_t>& starts) {
    Partition p;
    p.dim = csr.dim;
    p.row_begin = r0;
    p.local = r1 - r0;
    const int64_t D = csr.dim;
    int64_t max_up = -1, max_dn = -1;
    int64_t bnd_lo = 0, bnd_hi = 0;
    for (int64_t i = 0; i < p.local; ++i) {
        bool lo_ref = false, hi_ref = false;
        for (int64_t q = csr.offs[i]; q < csr.offs[i + 1]; ++q) {
            const int64_t g = csr.cols[q];
            if (g >= r0 && g < r1) continue;
            // ring distance above the range and below it decide the side
            const int64_t up = ((g - r1) % D + D) % D;
            const int64_t dn = ((r0 - 1 - g) % D + D) % D;
            if (up <= dn) {
                max_up = std::max(max_up, up);
                hi_ref = true;
            } else {
                max_dn = std::max(max_dn, dn);
                lo_ref = true;
            }
        }
        if (lo_ref) bnd_lo = i + 1;
        if (hi_ref) bnd_hi = std::max(bnd_hi, p.local - i);
    }
    auto owner = [&](int64_t g) {
        return static_cast<int>(std::upper_bound(starts.begin(), starts.end(), g) - starts.begin()) - 1;
    };
    if (max_up >= 0) {
        p.halo_hi = max_up + 1;
        p.hi_src_begin = r1 % D;
        p.hi_rank = owner(p.hi_src_begin);
        if (p.hi_src_begin + p.halo_hi > starts[p.hi_rank + 1])
            fail(CHEBFD_ERR_UNSUPPORTED, "upper halo spans more than one neighbour rank");
    }
    if (max_dn >= 0) {
        p.halo_lo = max_dn + 1;
        const int64_t lo_end = r0 == 0 ? D : r0;
        p.lo_src_begin = lo_end - p.halo_lo;
        p.lo_rank = owner(lo_end - 1);
        if (p.lo_src_begin < starts[p.lo_rank])
            fail(CHEBFD_ERR_UNSUPPORTED, "lower halo spans more than one neighbour rank");
    }
    p.bnd_lo = bnd_lo;
    p.bnd_hi = bnd_hi;
    if (p.bnd_lo + p.bnd_hi > p.local) {  // tiny partitions: every row is a boundary row
        p.bnd_lo = p.local;
        p.bnd_hi = 0;
    }
    return p;
}

Partition plan_rows_compact(const HostCsr& csr, int64_t r0, int64_t r1,
                            const std::vector<int64_t>& starts) {
    Partition p = plan_rows(csr, r0, r1, starts);
    const int64_t D = csr.dim;
    std::vector<int64_t> lo, hi, slo, shi;
    for (int64_t i = 0; i < p.local; ++i) {
        bool to_lo = false, to_hi = false;
        for (int64_t q = csr.offs[i]; q < csr.offs[i + 1]; ++q) {
            const int64_t g = csr.cols[q];
            if (g >= r0 && g < r1) continue;
            const int64_t up = ((g - r1) % D + D) % D;
            const int64_t dn = ((r0 - 1 - g) % D + D) % D;
            if (up <= dn) {
                hi.push_back(g);
                to_hi = true;
            } else {
                lo.push_back(g);
                to_lo = true;
            }
        }
        // structural symmetry: the rows that read a neighbour are the rows it reads
        if (to_lo) slo.push_back(i);
        if (to_hi) shi.push_back(i);
    }
    auto uniq = [](std::vector<int64_t>& v) {
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
    };
    uniq(lo);
    uniq(hi);
    p.compact = true;
    p.halo_lo_rows = std::move(lo);
    p.halo_hi_rows = std::move(hi);
    p.halo_lo = static_cast<int64_t>(p.halo_lo_rows.size());
    p.halo_hi = static_cast<int64_t>(p.halo_hi_rows.size());
    if (p.halo_lo) p.lo_src_begin = p.halo_lo_rows.front();
    if (p.halo_hi) p.hi_src_begin = p.halo_hi_rows.front();
    p.send_lo_rows = std::move(slo);
    p.send_hi_rows = std::move(shi);
    return p;
}

int64_t map_column(const Partition& p, int64_t g) {
    if (!p.compact) return colmap_of(p).map(g);
    if (g >= p.row_begin && g < p.row_begin + p.local) return g - p.row_begin + p.halo_lo;
    auto it = std::lower_bound(p.halo_lo_rows.begin(), p.halo_lo_rows.end(), g);
    if (it != p.halo_lo_rows.end() && *it == g) return it - p.halo_lo_rows.begin();
    it = std::lower_bound(p.halo_hi_rows.begin(), p.halo_hi_rows.end(), g);
    if (it != p.halo_hi_rows.end() && *it == g)
        return p.halo_lo + p.local + (it - p.halo_hi_rows.begin());
    return -2;
}

void plan_sends(Partition& p, int rank, int nranks, const int64_t* all) {
    if (p.compact) {
        // what a neighbour reads from us is what we read from it (structural symmetry);
        // the all-gathered halo sizes must agree with our send lists
        p.send_lo_n = p.lo_rank >= 0 && nranks > 1 ? static_cast<int64_t>(p.send_lo_rows.size()) : 0;
        p.send_hi_n = p.hi_rank >= 0 && nranks > 1 ? static_cast<int64_t>(p.send_hi_rows.size()) : 0;
        if (p.hi_rank >= 0 && nranks > 1 && all[4 * p.hi_rank + 2] == rank &&
            all[4 * p.hi_rank + 0] != p.send_hi_n)
            fail(CHEBFD_ERR_UNSUPPORTED, "compact halo: neighbour's request differs (structurally "
                                         "non-symmetric operator)");
        if (p.lo_rank >= 0 && nranks > 1 && all[4 * p.lo_rank + 3] == rank &&
            all[4 * p.lo_rank + 1] != p.send_lo_n)
            fail(CHEBFD_ERR_UNSUPPORTED, "compact halo: neighbour's request differs (structurally "
                                         "non-symmetric operator)");
        return;
    }
    // my hi neighbour's lo halo is my LAST rows; my lo neighbour's hi halo my FIRST rows
    if (p.hi_rank >= 0 && nranks > 1) {
        const int64_t need = all[4 * p.hi_rank + 0];
        if (all[4 * p.hi_rank + 2] == rank && need > 0) {
            p.send_hi_n = need;
            p.send_hi_begin = p.local - need;
        }
    }
    if (p.lo_rank >= 0 && nranks > 1) {
        const int64_t need = all[4 * p.lo_rank + 1];
        if (all[4 * p.lo_rank + 3] == rank && need > 0) {
            p.send_lo_n = need;
            p.send_lo_begin = 0;
        }
    }
    // a neighbour that needs rows from me although I do not read from it
    // (asymmetric stencils) is not supported by the symmetric protocol
    for (int q = 0; q < nranks; ++q) {
        if (q == rank) continue;
        if (all[4 * q + 2] == rank && all[4 * q + 0] > 0 && p.hi_rank != q)
            fail(CHEBFD_ERR_UNSUPPORTED, "asymmetric halo pattern");
        if (all[4 * q + 3] == rank && all[4 * q + 1] > 0 && p.lo_rank != q)
            fail(CHEBFD_ERR_UNSUPPORTED, "asymmetric halo pattern");
    }
    if (p.send_lo_n > p.local || p.send_hi_n > p.local)
        fail(CHEBFD_ERR_UNSUPPORTED, "neighbour halo larger than this rank's rows");
}

namespace {
void to_c(const Partition& p, chebfd_partition* o) {
    o->dim = p.dim;
    o->row_begin = p.row_begin;
    o->local_rows = p.local;
    o->halo_lo = p.halo_lo;
    o->halo_hi = p.halo_hi;
    o->lo_src_begin = p.lo_src_begin;
    o->hi_src_begin = p.hi_src_begin;
    o->lo_rank = p.lo_rank;
    o->hi_rank = p.hi_rank;
    o->bnd_lo = p.bnd_lo;
    o->bnd_hi = p.bnd_hi;
    o->send_lo_begin = p.send_lo_begin;
    o->send_lo_n = p.send_lo_n;
    o->send_hi_begin = p.send_hi_begin;
    o->send_hi_n = p.send_hi_n;
}
Partition from_c(const chebfd_partition* o) {
    Partition p;
    p.dim = o->dim;
    p.row_begin = o->row_begin;
    p.local = o->local_rows;
    p.halo_lo = o->halo_lo;
    p.halo_hi = o->halo_hi;
    p.lo_src_begin = o->lo_src_begin;
    p.hi_src_begin = o->hi_src_begin;
    p.lo_rank = o->lo_rank;
    p.hi_rank = o->hi_rank;
    p.bnd_lo = o->bnd_lo;
    p.bnd_hi = o->bnd_hi;
    p.send_lo_begin = o->send_lo_begin;
    p.send_lo_n = o->send_lo_n;
    p.send_hi_begin = o->send_hi_begin;
    p.send_hi_n = o->send_hi_n;
    return p;
}
}  // namespace

void lattice_starts(const chebfd_lattice& s, bool ti, int nranks, std::vector<int64_t>& starts) {
    const int64_t dim = ti ? 4 * s.lx * s.ly * s.lz : 2 * s.lx * s.ly;
    const int64_t plane = ti ? 4 * s.lx * s.ly : 2 * s.lx;  // TI z-plane / graphene y-row
    starts.assign(nranks + 1, 0);
    for (int q = 0; q < nranks; ++q) {
        int64_t a, b;
        plane_partition(dim, plane, q, nranks, &a, &b);
        starts[q] = a;
        starts[q + 1] = b;
    }
}

}  // namespace cfd

using namespace cfd;

extern "C" {

int chebfd_plan_partition(const chebfd_lattice* spec, int model, int rank, int nranks,
                          chebfd_partition* out) {
    return guard([&] {
        require(spec != nullptr && out != nullptr, "null argument");
        require(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank/nranks");
        require(model == 0 || model == 1, "model: 0 graphene, 1 topological insulator");
        const bool ti = model == 1;
        validate_lattice(*spec, ti);
        std::vector<int64_t> starts;
        lattice_starts(*spec, ti, nranks, starts);
        const int64_t r0 = starts[rank], r1 = starts[rank + 1];
        HostCsr csr = ti ? gen_topological_insulator(*spec, r0, r1) : gen_graphene(*spec, r0, r1);
        std::memset(out, 0, sizeof(*out));
        to_c(plan_rows(csr, r0, r1, starts), out);
    });
}

int chebfd_plan_sends(chebfd_partition* p, int rank, int nranks, const int64_t* all4) {
    return guard([&] {
        Partition q = from_c(p);
        plan_sends(q, rank, nranks, all4);
        to_c(q, p);
    });
}

int64_t chebfd_plan_map_column(const chebfd_partition* p, int64_t g) {
    return colmap_of(from_c(p)).map(g);
}

}  // extern "C"
