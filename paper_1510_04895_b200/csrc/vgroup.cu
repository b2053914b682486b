// Virtual rank groups: the distributed filter's P ranks driven in lockstep on ONE GPU.
//
// The multi-GPU path (capi.cu run_step_all) partitions the rows on lattice
// planes, exchanges the gathered operand's halo before each step and overlaps it with
// the interior rows, then reduces the dot partials of the interior and boundary
// launches in the last one.  Only one GPU is available to test it, and ranks whose
// kernels wait on one another must not run as separate launches on one GPU
// (B200_PROFILING.md).  A virtual group therefore runs all ranks as ONE stream-ordered
// program: each rank keeps its own Context (compute + comm stream, reduction scratch,
// SELL partition, blocks with halo rows), and one host thread enqueues every step for
// all ranks, in three phases per step:
//   1. each rank records the event that its gathered operand is produced;
//   2. each rank's comm stream waits for its own and its neighbours' producers and pulls
//      its halo rows straight from the neighbours' blocks (a gather kernel over the
//      neighbours' local row indices -- the P2P-pull form of the exchange);
//   3. each rank runs launch_split (interior rows concurrently with the pull, then the
//      boundary rows, cross-launch dot reduction) and its compute stream waits for the
//      neighbours' pulls before it may overwrite the buffer they read (the next step).
// No kernel waits on another; ordering is events between streams, so the whole
// sequence can be captured into one CUDA graph (fork from rank 0's stream, join back).
// Moments, dots and Gram matrices are summed over ranks in rank order on the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <tuple>
#include <vector>

#include "capi_common.hpp"

namespace cfd {

struct VGroup {
    int device = 0, P = 0;
    std::vector<Context*> ranks;
    std::vector<cudaEvent_t> ev_prod;  // per rank: the gathered operand is produced
    cudaEvent_t ev_join = nullptr;
    bool use_graphs = true;
    struct Graph {
        cudaGraphExec_t exec = nullptr;
        std::shared_ptr<DeviceBuffer> coeff;
        std::vector<std::shared_ptr<DeviceBuffer>> mom;
    };
    using Key = std::tuple<std::vector<const void*>, std::vector<const void*>, int, uint64_t,
                           uint64_t, bool, int64_t>;
    std::map<Key, Graph> graphs;
    DeviceBuffer coeff;
    std::vector<std::unique_ptr<DeviceBuffer>> mom;
    ~VGroup() {
        for (auto& kv : graphs)
            if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        for (auto e : ev_prod)
            if (e) cudaEventDestroy(e);
        if (ev_join) cudaEventDestroy(ev_join);
        mom.clear();
        for (Context* c : ranks) destroy_group_context(c);
    }
};

// drop the group's captured filters that reference matrix a or block storage x (called
// by purge_graphs when a rank's matrix or block is destroyed)
void vgroup_purge(VGroup& g, const void* a, const void* x) {
    for (auto it = g.graphs.begin(); it != g.graphs.end();) {
        const auto& as = std::get<0>(it->first);
        const auto& xs = std::get<1>(it->first);
        const bool hit = (a && std::find(as.begin(), as.end(), a) != as.end()) ||
                         (x && std::find(xs.begin(), xs.end(), x) != xs.end());
        if (hit) {
            if (it->second.exec) cudaGraphExecDestroy(it->second.exec);
            it = g.graphs.erase(it);
        } else {
            ++it;
        }
    }
}

namespace {

VGroup& group_of(chebfd_vgroup* g) {
    require(g != nullptr, "null virtual group");
    return *reinterpret_cast<VGroup*>(g);
}

// rank r's halo pull: lo / hi halo rows of `gathered` from the neighbours' blocks
void pull_halo(VGroup& g, const std::vector<const Matrix*>& A, const std::vector<Block*>& blk,
               int r) {
    Context& c = *g.ranks[r];
    const Matrix& a = *A[r];
    const Partition& p = a.part;
    Block& b = *blk[r];
    const int64_t rb = b.width * static_cast<int64_t>(b.scalar_bytes());
    char* base = static_cast<char*>(const_cast<void*>(gather_base(a, b)));
    if (p.lo_rank >= 0 && p.halo_lo > 0)
        launch_gather_rows(c, base, blk[p.lo_rank]->owned(), a.recv_lo_src.as<int64_t>(),
                           p.halo_lo, rb, c.comm_stream);
    if (p.hi_rank >= 0 && p.halo_hi > 0)
        launch_gather_rows(c, base + (p.halo_lo + p.local) * rb, blk[p.hi_rank]->owned(),
                           a.recv_hi_src.as<int64_t>(), p.halo_hi, rb, c.comm_stream);
}

// One step of every rank (same kind, rank-local arguments), lockstep.
void run_step_group(VGroup& g, const std::vector<const Matrix*>& A, std::vector<StepArgs> s,
                    const std::vector<Block*>& gathered) {
    const int P = g.P;
    for (int r = 0; r < P; ++r) {
        s[r].a = A[r];
        s[r].width_cols = gathered[r]->width;
        s[r].in = gather_base(*A[r], *gathered[r]);
    }
    // 1. producers
    for (int r = 0; r < P; ++r) CFD_CUDA(cudaEventRecord(g.ev_prod[r], g.ranks[r]->stream));
    // 2. halo pulls on the comm streams
    for (int r = 0; r < P; ++r) {
        Context& c = *g.ranks[r];
        const Partition& p = A[r]->part;
        CFD_CUDA(cudaStreamWaitEvent(c.comm_stream, g.ev_prod[r], 0));
        if (p.lo_rank >= 0) CFD_CUDA(cudaStreamWaitEvent(c.comm_stream, g.ev_prod[p.lo_rank], 0));
        if (p.hi_rank >= 0) CFD_CUDA(cudaStreamWaitEvent(c.comm_stream, g.ev_prod[p.hi_rank], 0));
        pull_halo(g, A, gathered, r);
        CFD_CUDA(cudaEventRecord(c.ev_b, c.comm_stream));
    }
    // 3. interior + boundary launches; then the neighbours' pulls must finish before this
    //    rank's next step overwrites the buffer they read
    for (int r = 0; r < P; ++r) {
        Context& c = *g.ranks[r];
        const Partition& p = A[r]->part;
        if (p.halo_lo == 0 && p.halo_hi == 0) {
            CFD_CUDA(cudaStreamWaitEvent(c.stream, c.ev_b, 0));
            StepArgs w = s[r];
            w.row0 = 0;
            w.row1 = p.local;
            w.partial_base = 0;
            w.final_launch = true;
            launch_step(c, w, c.stream);
        } else {
            launch_split(c, *A[r], s[r]);
        }
    }
    for (int r = 0; r < P; ++r) {
        Context& c = *g.ranks[r];
        const Partition& p = A[r]->part;
        if (p.lo_rank >= 0) CFD_CUDA(cudaStreamWaitEvent(c.stream, g.ranks[p.lo_rank]->ev_b, 0));
        if (p.hi_rank >= 0) CFD_CUDA(cudaStreamWaitEvent(c.stream, g.ranks[p.hi_rank]->ev_b, 0));
    }
}

std::vector<const Matrix*> matrices(VGroup& g, chebfd_matrix* const* a) {
    std::vector<const Matrix*> A(g.P);
    for (int r = 0; r < g.P; ++r) {
        A[r] = reinterpret_cast<const Matrix*>(a[r]);
        require(A[r] != nullptr && A[r]->ctx == g.ranks[r], "vgroup: matrix of another rank");
    }
    return A;
}

std::vector<Block*> blocks(VGroup& g, chebfd_block* const* b) {
    std::vector<Block*> B(g.P);
    for (int r = 0; r < g.P; ++r) {
        B[r] = reinterpret_cast<Block*>(b[r]);
        require(B[r] != nullptr && B[r]->ctx == g.ranks[r], "vgroup: block of another rank");
    }
    return B;
}

void sync_all(VGroup& g) {
    for (Context* c : g.ranks) ctx_sync(*c);
}

// fork every rank's stream from rank 0's (graph capture), join them back
void fork_all(VGroup& g) {
    Context& c0 = *g.ranks[0];
    CFD_CUDA(cudaEventRecord(g.ev_join, c0.stream));
    for (int r = 1; r < g.P; ++r) CFD_CUDA(cudaStreamWaitEvent(g.ranks[r]->stream, g.ev_join, 0));
}

void join_all(VGroup& g) {
    Context& c0 = *g.ranks[0];
    for (int r = 1; r < g.P; ++r) {
        CFD_CUDA(cudaEventRecord(g.ev_prod[r], g.ranks[r]->stream));
        CFD_CUDA(cudaStreamWaitEvent(c0.stream, g.ev_prod[r], 0));
    }
}

}  // namespace

}  // namespace cfd

using namespace cfd;

extern "C" {

int chebfd_vgroup_create(int device, int nranks, chebfd_vgroup** out) {
    return guard([&] {
        require(nranks >= 1 && out != nullptr, "vgroup_create: nranks must be >= 1");
        auto g = std::make_unique<VGroup>();
        g->device = device;
        g->P = nranks;
        for (int r = 0; r < nranks; ++r) {
            g->ranks.push_back(create_group_context(device, r, nranks));
            g->ranks.back()->vgroup = g.get();
            cudaEvent_t e;
            CFD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            g->ev_prod.push_back(e);
        }
        CFD_CUDA(cudaEventCreateWithFlags(&g->ev_join, cudaEventDisableTiming));
        *out = reinterpret_cast<chebfd_vgroup*>(g.release());
    });
}

int chebfd_vgroup_destroy(chebfd_vgroup* g) {
    return guard([&] {
        if (!g) return;
        VGroup* v = reinterpret_cast<VGroup*>(g);
        sync_all(*v);
        delete v;
    });
}

int chebfd_vgroup_context(chebfd_vgroup* g, int rank, chebfd_ctx** out) {
    return guard([&] {
        VGroup& v = group_of(g);
        require(rank >= 0 && rank < v.P, "vgroup_context: rank out of range");
        *out = reinterpret_cast<chebfd_ctx*>(v.ranks[rank]);
    });
}

int chebfd_vgroup_set_option(chebfd_vgroup* g, int option, int64_t value) {
    return guard([&] {
        VGroup& v = group_of(g);
        sync_all(v);
        for (auto& kv : v.graphs)
            if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        v.graphs.clear();
        if (option == CHEBFD_OPT_GRAPHS) {
            v.use_graphs = value != 0;
            return;
        }
        for (Context* c : v.ranks) {
            const int rc = chebfd_ctx_set_option(reinterpret_cast<chebfd_ctx*>(c), option, value);
            if (rc) fail(rc, g_last_error);
        }
    });
}

int chebfd_vgroup_matrix_lattice(chebfd_vgroup* g, int model, const chebfd_lattice* spec,
                                 chebfd_matrix** out) {
    return guard([&] {
        VGroup& v = group_of(g);
        require(spec != nullptr && out != nullptr, "vgroup_matrix_lattice: null argument");
        require(model == 0 || model == 1, "model: 0 graphene, 1 topological insulator");
        const bool ti = model == 1;
        validate_lattice(*spec, ti);
        std::vector<int64_t> starts;
        lattice_starts(*spec, ti, v.P, starts);
        std::vector<HostCsr> csr(v.P);
        std::vector<std::unique_ptr<Matrix>> m(v.P);
        int64_t nnz = 0;
        for (int r = 0; r < v.P; ++r) {
            Context& c = *v.ranks[r];
            csr[r] = ti ? gen_topological_insulator(*spec, starts[r], starts[r + 1])
                        : gen_graphene(*spec, starts[r], starts[r + 1]);
            nnz += static_cast<int64_t>(csr[r].cols.size());
            m[r] = std::make_unique<Matrix>();
            m[r]->ctx = &c;
            m[r]->kind = csr[r].kind;
            m[r]->nnz_local = static_cast<int64_t>(csr[r].cols.size());
            // both models are Hermitian: structurally symmetric, compact halos apply
            m[r]->part = c.compact_halo && v.P > 1
                             ? plan_rows_compact(csr[r], starts[r], starts[r + 1], starts)
                             : plan_rows(csr[r], starts[r], starts[r + 1], starts);
        }
        // what the NCCL path all-gathers: (halo_lo, halo_hi, lo_rank, hi_rank) of every rank
        std::vector<int64_t> all(4 * v.P);
        for (int r = 0; r < v.P; ++r) {
            const Partition& p = m[r]->part;
            all[4 * r + 0] = p.halo_lo;
            all[4 * r + 1] = p.halo_hi;
            all[4 * r + 2] = p.lo_rank;
            all[4 * r + 3] = p.hi_rank;
        }
        for (int r = 0; r < v.P; ++r) plan_sends(m[r]->part, r, v.P, all.data());
        for (int r = 0; r < v.P; ++r) {
            Context& c = *v.ranks[r];
            Matrix& mr = *m[r];
            mr.nnz_global = nnz;
            if (ti) {
                mr.plane_rows = 4 * spec->lx * spec->ly;
                mr.line_rows = 4 * spec->lx;
            }
            build_matrix_device(c, mr, csr[r]);
            mr.hermitian = true;
            // the neighbours' local indices of this rank's halo rows (pulled by rank r)
            const Partition& p = mr.part;
            auto src_list = [&](int q, bool lo) {
                std::vector<int64_t> idx;
                const int64_t n = lo ? p.halo_lo : p.halo_hi;
                for (int64_t i = 0; i < n; ++i) {
                    const int64_t gl = p.compact ? (lo ? p.halo_lo_rows[i] : p.halo_hi_rows[i])
                                                 : (lo ? p.lo_src_begin : p.hi_src_begin) + i;
                    idx.push_back(gl - starts[q]);
                }
                return idx;
            };
            auto up = [&](DeviceBuffer& d, const std::vector<int64_t>& h) {
                d.ensure(sizeof(int64_t) * std::max<size_t>(h.size(), 1));
                if (!h.empty())
                    CFD_CUDA(cudaMemcpyAsync(d.p, h.data(), sizeof(int64_t) * h.size(),
                                             cudaMemcpyHostToDevice, c.stream));
            };
            if (p.lo_rank >= 0) up(mr.recv_lo_src, src_list(p.lo_rank, true));
            if (p.hi_rank >= 0) up(mr.recv_hi_src, src_list(p.hi_rank, false));
            ctx_sync(c);
        }
        for (int r = 0; r < v.P; ++r) out[r] = reinterpret_cast<chebfd_matrix*>(m[r].release());
    });
}

int chebfd_vgroup_apply_filter(chebfd_vgroup* g, chebfd_matrix* const* a, chebfd_block* const* x,
                               const double* combined, int degree, double alpha, double beta,
                               double* moments) {
    return guard([&] {
        VGroup& v = group_of(g);
        const int P = v.P;
        auto A = matrices(v, a);
        auto X = blocks(v, x);
        if (degree < 2) fail(CHEBFD_ERR_INVALID_ARGUMENT, "apply_filter: degree must be >= 2");
        const bool want = moments != nullptr;
        const int64_t nb = X[0]->width;
        const bool dbl = want && moment_doubling(*v.ranks[0], *A[0]);
        std::vector<FilterWorkspace*> ws(P);
        for (int r = 0; r < P; ++r) {
            Context& c = *v.ranks[r];
            check_conforms(*A[r], *X[r], "apply_filter");
            require(X[r]->width == nb, "vgroup apply_filter: block widths differ");
            ws[r] = &filter_workspace(c, *A[r], nb, want && !dbl);
            Matrix& am = const_cast<Matrix&>(*A[r]);
            if (c.kernel_variant >= 1) {
                ensure_scaled_values(c, am, alpha, c.stream);
                ensure_scaled_values(c, am, 2.0 * alpha, c.stream);
                am.scaled_evicted = false;
            }
        }
        const size_t coeff_bytes = sizeof(double) * (degree + 1);
        const size_t mom_bytes = sizeof(double) * (degree + 1) * std::max<int64_t>(nb, 1);
        const size_t mom_alloc = mom_bytes + (dbl ? 3 * sizeof(double) * std::max<int64_t>(nb, 1) : 0);
        // the step sequence of every rank (identical kinds; rank-local buffers)
        auto enqueue = [&](const double* coeff_dev, const std::vector<double*>& mom_dev) {
            std::vector<std::vector<std::pair<StepArgs, Block*>>> steps(P);
            for (int r = 0; r < P; ++r)
                enqueue_filter(*v.ranks[r], *A[r], *X[r], degree, alpha, beta, coeff_dev,
                               mom_dev[r], *ws[r], [&](const StepArgs& s, Block& gb) {
                                   steps[r].emplace_back(s, &gb);
                               });
            for (size_t i = 0; i < steps[0].size(); ++i) {
                std::vector<StepArgs> s(P);
                std::vector<Block*> gb(P);
                for (int r = 0; r < P; ++r) {
                    require(steps[r].size() == steps[0].size(), "vgroup: ranks disagree on the steps");
                    s[r] = steps[r][i].first;
                    gb[r] = steps[r][i].second;
                }
                run_step_group(v, A, s, gb);
            }
        };
        sync_all(v);
        Context& c0 = *v.ranks[0];
        std::vector<double*> mom_dev(P, nullptr);
        if (v.use_graphs) {
            VGroup::Key key;
            for (int r = 0; r < P; ++r) {
                std::get<0>(key).push_back(A[r]);
                std::get<1>(key).push_back(X[r]->owned());
            }
            std::get<2>(key) = degree;
            std::memcpy(&std::get<3>(key), &alpha, 8);
            std::memcpy(&std::get<4>(key), &beta, 8);
            std::get<5>(key) = want;
            std::get<6>(key) = nb;
            auto it = v.graphs.find(key);
            if (it == v.graphs.end()) {
                VGroup::Graph e;
                e.coeff = std::make_shared<DeviceBuffer>(coeff_bytes);
                for (int r = 0; r < P; ++r) {
                    e.mom.push_back(want ? std::make_shared<DeviceBuffer>(mom_alloc) : nullptr);
                    mom_dev[r] = want ? e.mom[r]->as<double>() : nullptr;
                }
                CFD_CUDA(cudaMemcpyAsync(e.coeff->p, combined, coeff_bytes, cudaMemcpyHostToDevice,
                                         c0.stream));
                ctx_sync(c0);
                cudaGraph_t gr = nullptr;
                std::vector<int64_t> before(P);
                for (int r = 0; r < P; ++r) before[r] = v.ranks[r]->launches;
                CFD_CUDA(cudaStreamBeginCapture(c0.stream, cudaStreamCaptureModeThreadLocal));
                try {
                    fork_all(v);
                    enqueue(e.coeff->as<double>(), mom_dev);
                    join_all(v);
                } catch (...) {
                    cudaStreamEndCapture(c0.stream, &gr);
                    if (gr) cudaGraphDestroy(gr);
                    throw;
                }
                CFD_CUDA(cudaStreamEndCapture(c0.stream, &gr));
                CFD_CUDA(cudaGraphInstantiate(&e.exec, gr, 0));
                CFD_CUDA(cudaGraphDestroy(gr));
                it = v.graphs.emplace(key, e).first;
            } else {
                CFD_CUDA(cudaMemcpyAsync(it->second.coeff->p, combined, coeff_bytes,
                                         cudaMemcpyHostToDevice, c0.stream));
                for (int r = 0; r < P; ++r)
                    mom_dev[r] = want ? it->second.mom[r]->as<double>() : nullptr;
            }
            CFD_CUDA(cudaGraphLaunch(it->second.exec, c0.stream));
            ctx_sync(c0);
        } else {
            v.coeff.ensure(coeff_bytes);
            CFD_CUDA(cudaMemcpyAsync(v.coeff.p, combined, coeff_bytes, cudaMemcpyHostToDevice,
                                     c0.stream));
            ctx_sync(c0);
            v.mom.resize(P);
            for (int r = 0; r < P; ++r) {
                if (!want) continue;
                if (!v.mom[r]) v.mom[r] = std::make_unique<DeviceBuffer>();
                v.mom[r]->ensure(mom_alloc);
                mom_dev[r] = v.mom[r]->as<double>();
            }
            enqueue(v.coeff.as<double>(), mom_dev);
            sync_all(v);
        }
        if (want) {
            // allreduce in rank order
            const size_t n = static_cast<size_t>(degree + 1) * nb;
            std::vector<double> part(n);
            std::fill(moments, moments + n, 0.0);
            for (int r = 0; r < P; ++r) {
                CFD_CUDA(cudaMemcpy(part.data(), mom_dev[r], mom_bytes, cudaMemcpyDeviceToHost));
                for (size_t i = 0; i < n; ++i) moments[i] += part[i];
            }
            if (dbl) moments_from_doubling(moments, degree + 1, nb);
        }
    });
}

int chebfd_vgroup_spmmvm_fused(chebfd_vgroup* g, chebfd_matrix* const* a, chebfd_block* const* u,
                               chebfd_block* const* w, chebfd_block* const* x, double alpha,
                               double beta, double coeff, void* dots) {
    return guard([&] {
        VGroup& v = group_of(g);
        const int P = v.P;
        auto A = matrices(v, a);
        auto U = blocks(v, u);
        auto W = blocks(v, w);
        auto X = blocks(v, x);
        std::vector<StepArgs> s(P);
        const size_t bytes = static_cast<size_t>(U[0]->width) * U[0]->scalar_bytes();
        for (int r = 0; r < P; ++r) {
            Context& c = *v.ranks[r];
            check_same_shape(*U[r], *W[r]);
            check_same_shape(*U[r], *X[r]);
            check_conforms(*A[r], *U[r], "spmmvm_fused");
            if (U[r]->owned() == W[r]->owned() || U[r]->owned() == X[r]->owned() ||
                W[r]->owned() == X[r]->owned())
                fail(CHEBFD_ERR_INVALID_ARGUMENT, "spmmvm_fused: U, W, X must not alias");
            if (c.kernel_variant >= 1)
                ensure_scaled_values(c, const_cast<Matrix&>(*A[r]), 2.0 * alpha, c.stream);
            s[r] = StepArgs{};
            s[r].kind_step = kStepFused;
            s[r].w = W[r]->owned();
            s[r].x = X[r]->owned();
            s[r].alpha = 2.0 * alpha;
            s[r].beta = 2.0 * beta;
            s[r].c0 = coeff;
            s[r].dots_mode = dots ? 1 : 0;
            if (dots) {
                c.dscratch.ensure(bytes);
                s[r].dots_out = c.dscratch.p;
            }
        }
        sync_all(v);
        run_step_group(v, A, s, U);
        sync_all(v);
        if (dots) {
            std::vector<double> part(bytes / 8), tot(bytes / 8, 0.0);
            for (int r = 0; r < P; ++r) {
                CFD_CUDA(cudaMemcpy(part.data(), v.ranks[r]->dscratch.p, bytes, cudaMemcpyDeviceToHost));
                for (size_t i = 0; i < part.size(); ++i) tot[i] += part[i];
            }
            std::memcpy(dots, tot.data(), bytes);
        }
    });
}

int chebfd_vgroup_gram(chebfd_vgroup* g, chebfd_block* const* x, chebfd_block* const* y,
                       void* out) {
    return guard([&] {
        VGroup& v = group_of(g);
        auto X = blocks(v, x);
        auto Y = blocks(v, y);
        const size_t bytes = static_cast<size_t>(X[0]->width * Y[0]->width) * X[0]->scalar_bytes();
        std::vector<double> part(bytes / 8), tot(bytes / 8, 0.0);
        for (int r = 0; r < v.P; ++r) {
            Context& c = *v.ranks[r];
            require(X[r]->rows == Y[r]->rows && X[r]->kind == Y[r]->kind, "gram: dimension mismatch");
            c.dscratch.ensure(std::max<size_t>(bytes, 16));
            gemm_gram(c, *X[r], *Y[r], c.dscratch.p);
            CFD_CUDA(cudaMemcpyAsync(part.data(), c.dscratch.p, bytes, cudaMemcpyDeviceToHost, c.stream));
            ctx_sync(c);
            for (size_t i = 0; i < part.size(); ++i) tot[i] += part[i];
        }
        std::memcpy(out, tot.data(), bytes);
    });
}

int chebfd_vgroup_halo_rows(chebfd_matrix* a, int64_t* halo_lo, int64_t* halo_hi,
                            int64_t* send_lo, int64_t* send_hi) {
    return guard([&] {
        const Matrix& m = *reinterpret_cast<const Matrix*>(a);
        if (halo_lo) *halo_lo = m.part.halo_lo;
        if (halo_hi) *halo_hi = m.part.halo_hi;
        if (send_lo) *send_lo = m.part.send_lo_n;
        if (send_hi) *send_hi = m.part.send_hi_n;
    });
}

}  // extern "C"
