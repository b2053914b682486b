// extern "C" layer of chebfd_b200 (include/chebfd_b200.h): contexts, SELL
// matrices, device block vectors, the kernel entry points and apply_filter.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "internal.hpp"
#include "capi_common.hpp"

namespace cfd {

thread_local std::string g_last_error;

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(CHEBFD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void cublas_check(int st, const char* what) {
    if (st != 0) fail(CHEBFD_ERR_CUDA, std::string(what) + ": cuBLAS status " + std::to_string(st));
}

void nccl_check(int st, const char* what) {
    if (st != 0)
        fail(CHEBFD_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(static_cast<ncclResult_t>(st)));
}

DeviceBuffer::DeviceBuffer(size_t n) { ensure(n); }
DeviceBuffer::~DeviceBuffer() {
    if (p) cudaFree(p);
}
void DeviceBuffer::ensure(size_t n) {
    if (n <= bytes && p) return;
    if (p) CFD_CUDA(cudaFree(p));
    p = nullptr;
    bytes = 0;
    const size_t alloc = std::max<size_t>(n, 256);
    CFD_CUDA(cudaMalloc(&p, alloc));
    bytes = alloc;
}

void* Context::take_block_mem(size_t bytes) {
    auto it = block_cache.find(bytes);
    if (it != block_cache.end()) {
        void* p = it->second;
        block_cache.erase(it);
        block_cache_bytes -= bytes;
        return p;
    }
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        trim_block_cache();
        CFD_CUDA(cudaMalloc(&p, bytes));
    }
    return p;
}

void Context::give_block_mem(void* p, size_t bytes) {
    if (!p) return;
    if (bytes > block_cache_limit) {
        cudaFree(p);
        return;
    }
    while (block_cache_bytes + bytes > block_cache_limit && !block_cache.empty()) {
        auto it = std::prev(block_cache.end());  // drop the largest cached block
        block_cache_bytes -= it->first;
        cudaFree(it->second);
        block_cache.erase(it);
    }
    block_cache.emplace(bytes, p);
    block_cache_bytes += bytes;
}

void Context::trim_block_cache() {
    for (auto& kv : block_cache) cudaFree(kv.second);
    block_cache.clear();
    block_cache_bytes = 0;
}

Block::~Block() {
    if (ctx && buf.p) {
        ctx->give_block_mem(buf.p, buf.bytes);
        buf.p = nullptr;
        buf.bytes = 0;
    }
}

Context::~Context() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
    graphs.clear();
    filter_ws.clear();
    if (cublas) cublasDestroy(reinterpret_cast<cublasHandle_t>(cublas));
    destroy_cusolver(*this);
    if (nccl) ncclCommDestroy(nccl);
    for (auto& e : timers)
        if (e) cudaEventDestroy(e);
    if (ev_a) cudaEventDestroy(ev_a);
    if (ev_b) cudaEventDestroy(ev_b);
    if (stream) cudaStreamDestroy(stream);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    if (host_pinned) cudaFreeHost(host_pinned);
    trim_block_cache();
}

void* Context::pinned(size_t bytes) {
    if (bytes > host_pinned_bytes) {
        if (host_pinned) CFD_CUDA(cudaFreeHost(host_pinned));
        host_pinned = nullptr;
        const size_t n = std::max<size_t>(bytes, 1 << 16);
        CFD_CUDA(cudaMallocHost(&host_pinned, n));
        host_pinned_bytes = n;
    }
    return host_pinned;
}

// ---------------------------------------------------------- start blocks --
// BlockVector::randomize (block_vector.hpp:42-51) of this rank's rows: the
// reference's stream generated on the host (all threads) in pieces of one RNG
// chunk per thread, into two pinned buffers, each piece's upload overlapping
// the generation of the next.
void randomize_upload(Context& c, Block& b, uint64_t seed) {
    const int64_t count = b.rows * b.width;
    const size_t esz = b.kind ? 16 : 8;
    const int64_t first = b.row_begin * b.width;
    const int64_t kPiece = std::max<int64_t>(
        int64_t{1} << 22,
        std::min<int64_t>(NormalStream::parallel_piece(b.kind), (int64_t{1} << 30) / esz));
    if (count <= kPiece) {
        std::vector<double> h(static_cast<size_t>(count) * (b.kind ? 2 : 1));
        host_randomize(b.kind, seed, first, count, h.data());
        if (count)
            CFD_CUDA(cudaMemcpyAsync(b.owned(), h.data(), b.owned_bytes(), cudaMemcpyHostToDevice,
                                     c.stream));
        ctx_sync(c);
        return;
    }
    char* pin = static_cast<char*>(c.pinned(2 * kPiece * esz));
    cudaEvent_t done[2];
    CFD_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
    CFD_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
    NormalStream ns(seed);
    char* dev = static_cast<char*>(b.owned());
    try {
        for (int64_t off = 0, k = 0; off < count; off += kPiece, ++k) {
            const int buf = static_cast<int>(k & 1);
            const int64_t n = std::min(kPiece, count - off);
            char* h = pin + buf * kPiece * esz;
            if (k >= 2) CFD_CUDA(cudaEventSynchronize(done[buf]));
            ns.emit(b.kind, first + off, n, h);
            CFD_CUDA(cudaMemcpyAsync(dev + off * esz, h, n * esz, cudaMemcpyHostToDevice, c.stream));
            CFD_CUDA(cudaEventRecord(done[buf], c.stream));
        }
        ctx_sync(c);
    } catch (...) {
        cudaStreamSynchronize(c.stream);
        cudaEventDestroy(done[0]);
        cudaEventDestroy(done[1]);
        throw;
    }
    cudaEventDestroy(done[0]);
    cudaEventDestroy(done[1]);
}

// The same stream generated on a helper thread with its own CUDA stream and pinned
// buffers, so a solve's start block is produced while the device runs the Lanczos bounds
// and the KPM DOS (the block must not be touched until join()).
AsyncRandomize::AsyncRandomize(Context& c, Block& b, uint64_t seed) {
    const int device = c.device;
    th_ = std::thread([this, &b, seed, device] {
        cudaStream_t st = nullptr;
        char* pin = nullptr;
        cudaEvent_t done[2] = {nullptr, nullptr};
        try {
            CFD_CUDA(cudaSetDevice(device));
            CFD_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            const int64_t count = b.rows * b.width;
            const size_t esz = b.kind ? 16 : 8;
            const int64_t first = b.row_begin * b.width;
            const int64_t kPiece = std::max<int64_t>(
                int64_t{1} << 22,
                std::min<int64_t>(NormalStream::parallel_piece(b.kind), (int64_t{1} << 30) / esz));
            CFD_CUDA(cudaMallocHost(reinterpret_cast<void**>(&pin),
                                    2 * static_cast<size_t>(std::min(kPiece, std::max<int64_t>(count, 1))) * esz));
            CFD_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
            CFD_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
            NormalStream ns(seed);
            char* dev = static_cast<char*>(b.owned());
            const int64_t piece = std::min(kPiece, std::max<int64_t>(count, 1));
            for (int64_t off = 0, k = 0; off < count; off += piece, ++k) {
                if (cancel_.load(std::memory_order_relaxed)) break;  // block no longer wanted
                const int buf = static_cast<int>(k & 1);
                const int64_t n = std::min(piece, count - off);
                char* h = pin + buf * piece * esz;
                if (k >= 2) CFD_CUDA(cudaEventSynchronize(done[buf]));
                ns.emit(b.kind, first + off, n, h);
                CFD_CUDA(cudaMemcpyAsync(dev + off * esz, h, n * esz, cudaMemcpyHostToDevice, st));
                CFD_CUDA(cudaEventRecord(done[buf], st));
            }
            CFD_CUDA(cudaStreamSynchronize(st));
        } catch (...) {
            err_ = std::current_exception();
        }
        if (st) cudaStreamSynchronize(st);
        for (cudaEvent_t e : done)
            if (e) cudaEventDestroy(e);
        if (pin) cudaFreeHost(pin);
        if (st) cudaStreamDestroy(st);
    });
}

void AsyncRandomize::join() {
    if (th_.joinable()) th_.join();
    if (err_) {
        auto e = err_;
        err_ = nullptr;
        std::rethrow_exception(e);
    }
}

AsyncRandomize::~AsyncRandomize() {
    // not joined (an early return or an error before the block was needed): stop after the
    // piece in flight instead of generating the rest
    cancel_.store(true, std::memory_order_relaxed);
    if (th_.joinable()) th_.join();
}

// ---------------------------------------------------------------- helpers --
void ctx_sync(Context& c) { CFD_CUDA(cudaStreamSynchronize(c.stream)); }

void purge_graphs(Context& c, const void* a, const void* x) {
    if (c.vgroup) vgroup_purge(*c.vgroup, a, x);
    for (auto it = c.graphs.begin(); it != c.graphs.end();) {
        if ((a && it->first.a == a) || (x && it->first.x == x)) {
            cudaGraphExecDestroy(it->second.exec);
            it = c.graphs.erase(it);
        } else {
            ++it;
        }
    }
    if (a)
        for (auto it = c.filter_ws.begin(); it != c.filter_ws.end();) {
            if (std::get<0>(it->first) == a)
                it = c.filter_ws.erase(it);
            else
                ++it;
        }
}

std::unique_ptr<Block> make_block(Context& c, const Matrix* m, int kind, int64_t rows,
                                  int64_t width, bool zero) {
    require(width >= 0 && rows >= 0, "BlockVector: negative shape");
    auto b = std::make_unique<Block>();
    b->ctx = &c;
    b->kind = kind;
    b->rows = rows;
    b->width = width;
    b->shape_of = m;
    if (m) {
        b->halo_lo = m->part.halo_lo;
        b->halo_hi = m->part.halo_hi;
        b->row_begin = m->part.row_begin;
        b->dim_global = m->part.dim;
    } else {
        b->dim_global = rows;
    }
    const size_t bytes = static_cast<size_t>((b->halo_lo + rows + b->halo_hi) * width) *
                         b->scalar_bytes();
    b->buf.bytes = std::max<size_t>(bytes, 256);
    b->buf.p = c.take_block_mem(b->buf.bytes);
    if (zero) {
        CFD_CUDA(cudaMemsetAsync(b->buf.p, 0, b->buf.bytes, c.stream));
    } else {
        const size_t rb = static_cast<size_t>(width) * b->scalar_bytes();
        if (b->halo_lo) CFD_CUDA(cudaMemsetAsync(b->buf.p, 0, b->halo_lo * rb, c.stream));
        if (b->halo_hi)
            CFD_CUDA(cudaMemsetAsync(static_cast<char*>(b->owned()) + rows * rb, 0, b->halo_hi * rb,
                                     c.stream));
    }
    return b;
}

void check_same_shape(const Block& x, const Block& y) {
    if (x.rows != y.rows || x.width != y.width || x.kind != y.kind || x.ctx != y.ctx)
        fail(CHEBFD_ERR_INVALID_ARGUMENT, "block vector shape mismatch");
}

void check_conforms(const Matrix& a, const Block& x, const char* who) {
    if (x.kind != a.kind) fail(CHEBFD_ERR_INVALID_ARGUMENT, std::string(who) + ": scalar kind mismatch");
    if (x.rows != a.part.local || x.row_begin != a.part.row_begin || x.ctx != a.ctx)
        fail(CHEBFD_ERR_INVALID_ARGUMENT, std::string(who) + ": dimension mismatch");
    if (x.halo_lo < a.part.halo_lo || x.halo_hi < a.part.halo_hi)
        fail(CHEBFD_ERR_INVALID_ARGUMENT,
             std::string(who) + ": gathered block lacks halo storage (create it from the matrix)");
}

// extended-row base pointer that matches the matrix's column numbering
const void* gather_base(const Matrix& a, const Block& b) {
    return static_cast<const char*>(b.owned()) -
           a.part.halo_lo * b.width * static_cast<int64_t>(b.scalar_bytes());
}

// Fill the halos of `b` from the neighbours (NCCL point-to-point on `st`).
// Message order per rank: send A (my last rows -> hi's lo halo), send B (my
// first rows -> lo's hi halo), recv A (lo halo), recv B (hi halo); this
// matches in order even when lo and hi are the same peer (2-rank ring).
// Compact halos first gather the sent rows into contiguous pack buffers (one small kernel
// per side on `st`); the receiver's halo region is contiguous either way.
void ensure_halo_buffers(Context& c, Matrix& a, int64_t width) {
    const Partition& p = a.part;
    if (!p.compact || c.nranks == 1) return;
    const size_t rb = static_cast<size_t>(width) * (a.kind ? 16 : 8);
    a.pack_lo.ensure(std::max<size_t>(p.send_lo_n * rb, 16));
    a.pack_hi.ensure(std::max<size_t>(p.send_hi_n * rb, 16));
}

void exchange_halo(Context& c, const Matrix& a, Block& b, cudaStream_t st) {
    if (c.nranks == 1 || !c.nccl) return;
    const Partition& p = a.part;
    const size_t row_bytes = static_cast<size_t>(b.width) * b.scalar_bytes();
    const size_t words = row_bytes / 8;
    char* own = static_cast<char*>(b.owned());
    char* base = static_cast<char*>(const_cast<void*>(gather_base(a, b)));
    const char* send_hi = own + p.send_hi_begin * row_bytes;
    const char* send_lo = own + p.send_lo_begin * row_bytes;
    if (p.compact) {
        Matrix& am = const_cast<Matrix&>(a);
        if (am.pack_hi.bytes < p.send_hi_n * row_bytes || am.pack_lo.bytes < p.send_lo_n * row_bytes) {
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            CFD_CUDA(cudaStreamIsCapturing(st, &cs));
            if (cs != cudaStreamCaptureStatusNone)
                fail(CHEBFD_ERR_RUNTIME, "halo pack buffers not sized before graph capture");
            ensure_halo_buffers(c, am, b.width);
        }
        if (p.hi_rank >= 0 && p.send_hi_n > 0)
            launch_gather_rows(c, am.pack_hi.p, own, am.send_hi_idx.as<int64_t>(), p.send_hi_n,
                               static_cast<int64_t>(row_bytes), st);
        if (p.lo_rank >= 0 && p.send_lo_n > 0)
            launch_gather_rows(c, am.pack_lo.p, own, am.send_lo_idx.as<int64_t>(), p.send_lo_n,
                               static_cast<int64_t>(row_bytes), st);
        send_hi = static_cast<const char*>(am.pack_hi.p);
        send_lo = static_cast<const char*>(am.pack_lo.p);
    }
    nccl_check(ncclGroupStart(), "ncclGroupStart");
    if (p.hi_rank >= 0 && p.send_hi_n > 0)
        nccl_check(ncclSend(send_hi, p.send_hi_n * words, ncclFloat64, p.hi_rank, c.nccl, st),
                   "ncclSend");
    if (p.lo_rank >= 0 && p.send_lo_n > 0)
        nccl_check(ncclSend(send_lo, p.send_lo_n * words, ncclFloat64, p.lo_rank, c.nccl, st),
                   "ncclSend");
    if (p.lo_rank >= 0 && p.halo_lo > 0)
        nccl_check(ncclRecv(base, p.halo_lo * words, ncclFloat64, p.lo_rank, c.nccl, st),
                   "ncclRecv");
    if (p.hi_rank >= 0 && p.halo_hi > 0)
        nccl_check(ncclRecv(base + (p.halo_lo + p.local) * row_bytes, p.halo_hi * words,
                            ncclFloat64, p.hi_rank, c.nccl, st), "ncclRecv");
    nccl_check(ncclGroupEnd(), "ncclGroupEnd");
}

void allreduce_sum(Context& c, double* dev, size_t n, cudaStream_t st) {
    if (c.nranks == 1 || !c.nccl || n == 0) return;
    nccl_check(ncclAllReduce(dev, dev, n, ncclFloat64, ncclSum, c.nccl, st), "ncclAllReduce");
}

// One Chebyshev-type step over all owned rows, with the halo exchange of the
// gathered operand overlapped with the interior rows when distributed.
void run_step_all(Context& c, const Matrix& a, StepArgs s, Block& gathered) {
    if (c.kernel_variant >= 1 && s.alpha != 1.0) {
        // the TMA step kernel reads values pre-multiplied by alpha; build the
        // copy now unless a graph is being captured (apply_filter pre-builds)
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        CFD_CUDA(cudaStreamIsCapturing(c.stream, &cs));
        if (cs == cudaStreamCaptureStatusNone) {
            Matrix& am = const_cast<Matrix&>(a);
            ensure_scaled_values(c, am, s.alpha, c.stream);
            if (am.scaled_evicted) {
                purge_graphs(c, &a, nullptr);
                am.scaled_evicted = false;
            }
        }
    }
    s.a = &a;
    s.width_cols = gathered.width;
    s.in = gather_base(a, gathered);
    const Partition& p = a.part;
    if (c.vgroup && (p.halo_lo || p.halo_hi))
        fail(CHEBFD_ERR_UNSUPPORTED, "a virtual-group rank's halo needs the chebfd_vgroup_* entry points");
    if (c.nranks == 1 || !c.nccl || (p.halo_lo == 0 && p.halo_hi == 0)) {
        s.row0 = 0;
        s.row1 = p.local;
        s.partial_base = 0;
        s.final_launch = true;
        s.pdl_ok = true;  // one kernel per step, stream-ordered after the previous one
        launch_step(c, s, c.stream);
        return;
    }
    // fork: comm stream waits for the producer of `gathered`
    CFD_CUDA(cudaEventRecord(c.ev_a, c.stream));
    CFD_CUDA(cudaStreamWaitEvent(c.comm_stream, c.ev_a, 0));
    exchange_halo(c, a, gathered, c.comm_stream);
    CFD_CUDA(cudaEventRecord(c.ev_b, c.comm_stream));
    launch_split(c, a, s);
}

// The step's launches once its halo exchange is enqueued on the comm stream and c.ev_b
// marks its completion: interior rows (no halo reads) concurrently with the exchange,
// then the boundary rows; the dot partials of the 2-3 launches are reduced by the last.
void launch_split(Context& c, const Matrix& a, StepArgs s) {
    Partition p = a.part;
    // lattice operators: widen the boundary regions to whole planes (rows that merely
    // could run early wait for the halo -- always safe), so every launch covers whole
    // planes and the band tile order applies to all of them
    if (a.plane_rows > 0 && p.local % a.plane_rows == 0) {
        const int64_t P = a.plane_rows;
        p.bnd_lo = std::min(p.local, (p.bnd_lo + P - 1) / P * P);
        p.bnd_hi = std::min(p.local - p.bnd_lo, (p.bnd_hi + P - 1) / P * P);
    }
    int used = 0, base = 0;
    // dot partials of column-slabbed launches cannot be split over interior and boundary
    // launches: such steps wait for the halo and run as one launch per slab
    StepArgs whole = s;
    whole.row0 = 0;
    whole.row1 = p.local;
    if (s.dots_mode != 0 && step_slab_count(c, whole) > 1) {
        CFD_CUDA(cudaStreamWaitEvent(c.stream, c.ev_b, 0));
        whole.partial_base = 0;
        whole.final_launch = true;
        launch_step(c, whole, c.stream);
        return;
    }
    const bool overlap = c.overlap;
    if (!overlap) CFD_CUDA(cudaStreamWaitEvent(c.stream, c.ev_b, 0));
    // interior rows (no halo reads)
    s.row0 = p.bnd_lo;
    s.row1 = p.local - p.bnd_hi;
    s.partial_base = 0;
    s.final_launch = false;
    s.grid_used = &used;
    if (s.row1 > s.row0) {
        launch_step(c, s, c.stream);
        base += used;
    }
    if (overlap) CFD_CUDA(cudaStreamWaitEvent(c.stream, c.ev_b, 0));
    // boundary rows
    if (p.bnd_lo > 0) {
        s.row0 = 0;
        s.row1 = p.bnd_lo;
        s.partial_base = base;
        s.final_launch = p.bnd_hi == 0;
        launch_step(c, s, c.stream);
        base += used;
    }
    if (p.bnd_hi > 0) {
        s.row0 = p.local - p.bnd_hi;
        s.row1 = p.local;
        s.partial_base = base;
        s.final_launch = true;
        launch_step(c, s, c.stream);
    }
    if (p.bnd_lo == 0 && p.bnd_hi == 0 && s.dots_mode) {
        // no boundary launch: reduce with a final empty-range launch
        s.row0 = s.row1 = 0;
        s.partial_base = base;
        s.final_launch = true;
        launch_step(c, s, c.stream);
    }
}

// ------------------------------------------------------ partition set-up --
// Derive halos of rows [r0, r1) from the global column indices they use
// (ring distance decides lo vs hi), then tell every rank what its
// neighbours need from it.
void setup_partition(Context& c, Matrix& m, const HostCsr& csr, int64_t r0, int64_t r1,
                     const std::vector<int64_t>& starts, bool compact) {
    m.part = compact && c.nranks > 1 ? plan_rows_compact(csr, r0, r1, starts)
                                     : plan_rows(csr, r0, r1, starts);
    Partition& p = m.part;
    const int P = c.nranks;
    // what do the neighbours need from me?  all-gather (halo_lo, halo_hi, lo_rank, hi_rank)
    std::vector<int64_t> mine = {p.halo_lo, p.halo_hi, p.lo_rank, p.hi_rank};
    std::vector<int64_t> all(4 * P, 0);
    if (P > 1) {
        DeviceBuffer d(sizeof(int64_t) * 4 * P);
        CFD_CUDA(cudaMemcpyAsync(d.as<int64_t>() + 4 * c.rank, mine.data(), sizeof(int64_t) * 4,
                                 cudaMemcpyHostToDevice, c.stream));
        nccl_check(ncclAllGather(d.as<int64_t>() + 4 * c.rank, d.p, 4, ncclInt64, c.nccl, c.stream),
                   "ncclAllGather");
        CFD_CUDA(cudaMemcpyAsync(all.data(), d.p, sizeof(int64_t) * 4 * P, cudaMemcpyDeviceToHost,
                                 c.stream));
        ctx_sync(c);
    } else {
        all = mine;
    }
    plan_sends(p, c.rank, P, all.data());
}

std::unique_ptr<Matrix> matrix_from_host_csr(Context& c, const HostCsr& csr, int64_t r0, int64_t r1,
                                             const std::vector<int64_t>& starts, int64_t nnz_global,
                                             bool symmetric, int64_t plane_rows = 0,
                                             int64_t line_rows = 0) {
    auto m = std::make_unique<Matrix>();
    m->ctx = &c;
    m->plane_rows = plane_rows;  // known before the build: the grouped form tiles by lines
    m->line_rows = line_rows;
    m->kind = csr.kind;
    m->nnz_local = static_cast<int64_t>(csr.cols.size());
    m->nnz_global = nnz_global;
    setup_partition(c, *m, csr, r0, r1, starts, symmetric && c.compact_halo);
    build_matrix_device(c, *m, csr);
    return m;
}

// Upload this rank's CSR (columns pre-mapped to extended rows for compact halos) and
// convert it to SELL on the device; upload the compact halo send lists.
void build_matrix_device(Context& c, Matrix& mat, const HostCsr& csr) {
    Matrix* m = &mat;
    const Partition& part = m->part;
    const int64_t rows = part.local, nnz = m->nnz_local;
    std::vector<int64_t> mapped;
    const int64_t* cols_h = csr.cols.data();
    if (part.compact) {
        mapped.resize(csr.cols.size());
        for (size_t q = 0; q < csr.cols.size(); ++q) {
            mapped[q] = map_column(part, csr.cols[q]);
            if (mapped[q] < 0) fail(CHEBFD_ERR_UNSUPPORTED, "matrix column outside this rank's rows and halos");
        }
        cols_h = mapped.data();
        auto up = [&](DeviceBuffer& d, const std::vector<int64_t>& v) {
            d.ensure(sizeof(int64_t) * std::max<size_t>(v.size(), 1));
            if (!v.empty())
                CFD_CUDA(cudaMemcpyAsync(d.p, v.data(), sizeof(int64_t) * v.size(),
                                         cudaMemcpyHostToDevice, c.stream));
        };
        up(m->send_lo_idx, part.send_lo_rows);
        up(m->send_hi_idx, part.send_hi_rows);
    }
    // upload the CSR of owned rows and convert on the device
    DeviceBuffer d_offs(sizeof(int64_t) * (rows + 1));
    DeviceBuffer d_cols(sizeof(int64_t) * std::max<int64_t>(nnz, 1));
    DeviceBuffer d_vals((csr.kind ? 16 : 8) * std::max<int64_t>(nnz, 1));
    CFD_CUDA(cudaMemcpyAsync(d_offs.p, csr.offs.data(), sizeof(int64_t) * (rows + 1),
                             cudaMemcpyHostToDevice, c.stream));
    if (nnz) {
        CFD_CUDA(cudaMemcpyAsync(d_cols.p, cols_h, sizeof(int64_t) * nnz,
                                 cudaMemcpyHostToDevice, c.stream));
        CFD_CUDA(cudaMemcpyAsync(d_vals.p, csr.vals.data(), sizeof(double) * csr.vals.size(),
                                 cudaMemcpyHostToDevice, c.stream));
    }
    build_sell(c, *m, d_offs.as<int64_t>(), d_cols.as<int64_t>(), d_vals.p, c.stream);
    ctx_sync(c);
}

int64_t allreduce_count(Context& c, int64_t v) {
    if (c.nranks == 1) return v;
    DeviceBuffer d(sizeof(int64_t));
    CFD_CUDA(cudaMemcpyAsync(d.p, &v, sizeof(int64_t), cudaMemcpyHostToDevice, c.stream));
    nccl_check(ncclAllReduce(d.p, d.p, 1, ncclInt64, ncclSum, c.nccl, c.stream), "ncclAllReduce");
    int64_t out = 0;
    CFD_CUDA(cudaMemcpyAsync(&out, d.p, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    ctx_sync(c);
    return out;
}

std::unique_ptr<Matrix> lattice_matrix(Context& c, const chebfd_lattice& s, bool ti) {
    validate_lattice(s, ti);
    std::vector<int64_t> starts;
    lattice_starts(s, ti, c.nranks, starts);
    const int64_t r0 = starts[c.rank], r1 = starts[c.rank + 1];
    HostCsr csr = ti ? gen_topological_insulator(s, r0, r1) : gen_graphene(s, r0, r1);
    const int64_t nnz_g = allreduce_count(c, static_cast<int64_t>(csr.cols.size()));
    // both models add every hopping with its conjugate (models.cpp:80-178): Hermitian,
    // hence structurally symmetric (compact halos apply)
    // TI: row = 4 (x + Lx (y + Ly z)) + orbital (models.hpp:15-19)
    auto m = matrix_from_host_csr(c, csr, r0, r1, starts, nnz_g, true, ti ? 4 * s.lx * s.ly : 0,
                                  ti ? 4 * s.lx : 0);
    m->hermitian = true;
    return m;
}

// --------------------------------------------------------- apply_filter --
// Fused steps n and n+1 in one wavefront launch where it applies (pair.cu):
// single-rank operators (no halo exchange between the steps), no dots.
bool run_pair_step(Context& c, const Matrix& a, Block& u, Block& w, Block& x, double alpha,
                   double beta, const double* coeff_dev, int n, void* x0, double* mom) {
    if (c.pair_mode == 0 || c.kernel_variant < 1) return false;
    if (a.part.halo_lo != 0 || a.part.halo_hi != 0) return false;
    StepArgs s{};
    s.kind_step = kStepFused;
    s.a = &a;
    s.width_cols = u.width;
    s.in = gather_base(a, u);
    s.w = w.owned();
    s.x = x.owned();
    s.x0 = x0;
    s.alpha = 2.0 * alpha;
    s.beta = 2.0 * beta;
    s.coeff_dev = coeff_dev;
    s.coeff_index = n;
    s.dots_mode = mom ? 2 : 0;
    s.dots_out = mom;
    s.row0 = 0;
    s.row1 = a.part.local;
    s.partial_base = 0;
    s.final_launch = true;
    return launch_step_pair(c, s, c.stream);
}

FilterWorkspace& filter_workspace(Context& c, const Matrix& a, int64_t width, bool moments) {
    auto key = std::make_tuple(static_cast<const void*>(&a), width, a.kind);
    FilterWorkspace& ws = c.filter_ws[key];
    if (!ws.u) ws.u = make_block(c, &a, a.kind, a.part.local, width, false);
    if (!ws.w) ws.w = make_block(c, &a, a.kind, a.part.local, width, false);
    if (moments && !ws.x0) ws.x0 = make_block(c, &a, a.kind, a.part.local, width, false);
    return ws;
}

// Enqueue apply_filter (filter.hpp:73-116) on c.stream.  coeff_dev holds
// combined[0..degree]; mom_dev (if moments) (degree+1) x width doubles.
bool moment_doubling(const Context& c, const Matrix& a) { return c.moments_mode == 1 && a.hermitian; }

void enqueue_filter(Context& c, const Matrix& a, Block& x, int degree, double alpha, double beta,
                    const double* coeff_dev, double* mom_dev, FilterWorkspace& ws) {
    enqueue_filter(c, a, x, degree, alpha, beta, coeff_dev, mom_dev, ws,
                   [&](const StepArgs& s, Block& g) { run_step_all(c, a, s, g); });
    if (mom_dev) allreduce_sum(c, mom_dev, static_cast<size_t>((degree + 1) * x.width), c.stream);
}

void enqueue_filter(Context& c, const Matrix& a, Block& x, int degree, double alpha, double beta,
                    const double* coeff_dev, double* mom_dev, FilterWorkspace& ws,
                    const std::function<void(const StepArgs&, Block&)>& run) {
    const bool moments = mom_dev != nullptr;
    // doubling (DMODE 4): step n's registers give the raw sums of moments 2n-2, 2n-1, so
    // only steps n <= degree/2 + 1 reduce and no x0 copy is kept (mom_dev has 2 spare rows)
    const bool dbl = moments && moment_doubling(c, a);
    const int64_t nb = x.width;
    // u = (alpha A + beta) x   [+ x0 = x (direct mode), m0 = <x,x>, m1 = <x,u>]
    StepArgs s{};
    s.kind_step = kStepSpmmvm;
    s.w = ws.u->owned();
    s.x0 = moments && !dbl ? ws.x0->owned() : nullptr;
    s.alpha = alpha;
    s.beta = beta;
    s.dots_mode = moments ? (dbl ? 4 : 3) : 0;
    s.dots_out = mom_dev;
    run(s, x);
    // w = 2(alpha A + beta)u - x;  x = g0c0 x + g1c1 u + g2c2 w   [+ m2 = <x0,w>; doubling:
    // raw <u,u>, <u,w> for m2, m3]
    StepArgs s2{};
    s2.kind_step = kStepStart2;
    s2.w = ws.w->owned();
    s2.x = x.owned();
    s2.alpha = 2.0 * alpha;
    s2.beta = 2.0 * beta;
    s2.coeff_dev = coeff_dev;
    s2.dots_mode = moments ? (dbl ? 4 : 2) : 0;
    s2.dots_out = moments ? mom_dev + 2 * nb : nullptr;
    run(s2, *ws.u);
    Block* pu = ws.u.get();
    Block* pw = ws.w.get();
    // delayed X update (CHEBFD_OPT_DELAYED_X = G): of each group of G steps the first G-1 run
    // without touching X (kStepRecur) and the last adds all their terms in the reference's
    // order (kStepFusedX2 / X3: the V's of the group are its registers' wi, ui, wn), so X is
    // read and written once per G steps -- same bits
    // launch-bound operators with doubling moments: pairs (fewer reducing steps per group
    // of work; C1 with moments 3.21 ms for pairs vs 3.29 ms for triples)
    const bool small = a.part.local / 64 < 4 * static_cast<int64_t>(c.num_sms);
    const int group = std::clamp(dbl && small && c.delayed_x == 3 ? 2 : c.delayed_x, 1, 3);
    int grp_pos = 0, grp_len = 1;
    for (int n = 3; n <= degree; ++n) {
        std::swap(pu, pw);  // swap handles, never copies
        if (grp_pos == 0) grp_len = std::min(group, degree - n + 1);
        const bool x_pending = grp_pos > 0;
        // the (opt-in) pair kernel carries direct <x0, w> moments only
        const bool dots_n = moments && !dbl;
        if (!x_pending && n < degree && !(moments && dbl && 2 * n - 3 <= degree) &&
            run_pair_step(c, a, *pu, *pw, x, alpha, beta, coeff_dev, n,
                          dots_n ? ws.x0->owned() : nullptr,
                          dots_n ? mom_dev + static_cast<int64_t>(n) * nb : nullptr)) {
            // steps n and n+1 done: W holds V_n, U holds V_{n+1} -- the roles after step n+1
            std::swap(pu, pw);
            ++n;
            continue;
        }
        StepArgs f{};
        // moments: direct <x0, V_n> in every step; doubling: a V_n-only step holds
        // V_{n-2}, V_{n-1}, V_n and yields moments 2n-3 .. 2n (mode 5), so the X-update
        // steps reduce nothing; a plain fused step yields 2n-2, 2n-1 (mode 4)
        int dmode = 0;
        int64_t mrow = n;
        if (grp_len > 1 && grp_pos == grp_len - 1) {
            // X += c_{n-2} V_{n-2} (X3 only), c_{n-1} V_{n-1}, c_n V_n
            f.kind_step = grp_len == 3 ? kStepFusedX3 : kStepFusedX2;
            grp_pos = 0;
            if (moments && !dbl) dmode = 2;
        } else if (grp_len > 1) {
            f.kind_step = kStepRecur;  // V_n only; its X term rides on the group's last step
            if (moments && !dbl) dmode = 2;
            if (dbl && grp_pos == 0 && 2 * n - 3 <= degree) {
                dmode = 5;  // moments 2n-3 .. 2n
                mrow = 2 * n - 3;
            } else if (dbl && grp_pos == 1 && 2 * n - 1 <= degree) {
                dmode = 6;  // the second V_n-only step of a triple adds 2n-1, 2n
                mrow = 2 * n - 1;
            }
            ++grp_pos;
        } else {
            f.kind_step = kStepFused;
            if (moments && !dbl) dmode = 2;
            if (dbl && 2 * n - 2 <= degree) {
                dmode = 4;
                mrow = 2 * n - 2;
            }
        }
        f.w = pw->owned();
        f.x = x.owned();
        f.x0 = dmode == 2 ? ws.x0->owned() : nullptr;
        f.alpha = 2.0 * alpha;  // kernel multiplies values by (2 alpha) as kernels.hpp:95
        f.beta = 2.0 * beta;
        f.coeff_dev = coeff_dev;
        f.coeff_index = n;
        f.dots_mode = dmode;
        f.dots_out = dmode ? mom_dev + mrow * nb : nullptr;
        run(f, *pu);
    }
}

void apply_filter_device(Context& c, const Matrix& a, Block& x, const double* combined, int degree,
                         double alpha, double beta, double* moments_host) {
    check_conforms(a, x, "apply_filter");
    if (degree < 2) fail(CHEBFD_ERR_INVALID_ARGUMENT, "apply_filter: degree must be >= 2");
    const bool moments = moments_host != nullptr;
    const bool dbl = moments && moment_doubling(c, a);
    const int64_t nb = x.width;
    FilterWorkspace& ws = filter_workspace(c, a, nb, moments && !dbl);
    Matrix& am = const_cast<Matrix&>(a);
    ensure_halo_buffers(c, am, nb);
    if (c.kernel_variant >= 1) {  // pre-scaled values for the start step (alpha) and 2 alpha steps
        ensure_scaled_values(c, am, alpha, c.stream);
        ensure_scaled_values(c, am, 2.0 * alpha, c.stream);
        if (am.scaled_evicted) {
            purge_graphs(c, &a, nullptr);
            am.scaled_evicted = false;
        }
    }
    GraphKey key{&a, x.owned(), degree, 0, 0, moments, nb};
    std::memcpy(&key.alpha_bits, &alpha, 8);
    std::memcpy(&key.beta_bits, &beta, 8);
    const size_t coeff_bytes = sizeof(double) * (degree + 1);
    const size_t mom_bytes = sizeof(double) * (degree + 1) * std::max<int64_t>(nb, 1);
    // doubling writes raw sums of 2 or 4 consecutive moments: up to three rows past the table
    const size_t mom_alloc = mom_bytes + (dbl ? 3 * sizeof(double) * std::max<int64_t>(nb, 1) : 0);
    auto finish_moments = [&] {
        if (dbl) moments_from_doubling(moments_host, degree + 1, nb);
    };
    if (c.use_graphs) {
        auto it = c.graphs.find(key);
        if (it == c.graphs.end()) {
            GraphEntry e;
            e.coeff = std::make_shared<DeviceBuffer>(coeff_bytes);
            if (moments) e.moments = std::make_shared<DeviceBuffer>(mom_alloc);
            CFD_CUDA(cudaMemcpyAsync(e.coeff->p, combined, coeff_bytes, cudaMemcpyHostToDevice,
                                     c.stream));
            e.coeff_host.assign(combined, combined + degree + 1);
            ctx_sync(c);
            cudaGraph_t g;
            const int64_t before = c.launches;
            CFD_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
            try {
                enqueue_filter(c, a, x, degree, alpha, beta, e.coeff->as<double>(),
                               moments ? e.moments->as<double>() : nullptr, ws);
            } catch (...) {
                cudaStreamEndCapture(c.stream, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            CFD_CUDA(cudaStreamEndCapture(c.stream, &g));
            e.kernels = c.launches - before;
            c.launches = before;
            CFD_CUDA(cudaGraphInstantiate(&e.exec, g, 0));
            CFD_CUDA(cudaGraphDestroy(g));
            it = c.graphs.emplace(key, e).first;
        } else if (!std::equal(combined, combined + degree + 1, it->second.coeff_host.begin())) {
            CFD_CUDA(cudaMemcpyAsync(it->second.coeff->p, combined, coeff_bytes,
                                     cudaMemcpyHostToDevice, c.stream));
            it->second.coeff_host.assign(combined, combined + degree + 1);
        }
        CFD_CUDA(cudaGraphLaunch(it->second.exec, c.stream));
        c.launches += it->second.kernels;
        if (moments) {
            CFD_CUDA(cudaMemcpyAsync(moments_host, it->second.moments->p, mom_bytes,
                                     cudaMemcpyDeviceToHost, c.stream));
            ctx_sync(c);
            finish_moments();
        }
        return;
    }
    c.coeffs.ensure(coeff_bytes);
    CFD_CUDA(cudaMemcpyAsync(c.coeffs.p, combined, coeff_bytes, cudaMemcpyHostToDevice, c.stream));
    double* mom_dev = nullptr;
    if (moments) {
        c.dscratch.ensure(mom_alloc);
        mom_dev = c.dscratch.as<double>();
    }
    enqueue_filter(c, a, x, degree, alpha, beta, c.coeffs.as<double>(), mom_dev, ws);
    if (moments) {
        CFD_CUDA(cudaMemcpyAsync(moments_host, mom_dev, mom_bytes, cudaMemcpyDeviceToHost, c.stream));
        ctx_sync(c);
        finish_moments();
    }
}

// ------------------------------------------------------ small reductions --
// column dots <x_k, y_k> summed over ranks -> host (S[nb])
void column_dots_host(Context& c, const Block& x, const Block& y, void* out) {
    check_same_shape(x, y);
    const size_t bytes = static_cast<size_t>(x.width) * x.scalar_bytes();
    c.dscratch.ensure(bytes);
    launch_column_reduce(c, x, y, 0, c.dscratch.p, c.stream);
    allreduce_sum(c, c.dscratch.as<double>(), bytes / 8, c.stream);
    CFD_CUDA(cudaMemcpyAsync(out, c.dscratch.p, bytes, cudaMemcpyDeviceToHost, c.stream));
    ctx_sync(c);
}

void gram_host(Context& c, const Block& x, const Block& y, void* out, bool herm) {
    if (x.rows != y.rows || x.kind != y.kind)
        fail(CHEBFD_ERR_INVALID_ARGUMENT, "gram: dimension mismatch");
    const int64_t nx = x.width, ny = y.width;
    const size_t bytes = static_cast<size_t>(nx * ny) * x.scalar_bytes();
    c.dscratch.ensure(std::max<size_t>(bytes, 16));
    gemm_gram(c, x, y, c.dscratch.p, herm);
    allreduce_sum(c, c.dscratch.as<double>(), bytes / 8, c.stream);
    CFD_CUDA(cudaMemcpyAsync(out, c.dscratch.p, bytes, cudaMemcpyDeviceToHost, c.stream));
    ctx_sync(c);
}

}  // namespace cfd

using namespace cfd;

// ============================================================== C ABI ==
extern "C" {

const char* chebfd_last_error(void) { return g_last_error.c_str(); }
const char* chebfd_version(void) { return "chebfd_b200 0.2 (sm_100a)"; }

int chebfd_build_features(void) { return CFD_EXPERIMENTAL ? CHEBFD_FEATURE_EXPERIMENTAL : 0; }

int chebfd_nccl_unique_id(unsigned char id[128]) {
    return guard([&] {
        ncclUniqueId u;
        nccl_check(ncclGetUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, u.internal, 128);
    });
}

// One CUDA device per process (one process per GPU, torchrun-style): entry points launch
// on the thread's current device and the kernel attribute / occupancy caches are keyed by
// kernel only, so contexts on two devices in one process are refused.
static std::mutex g_dev_mu;
static int g_dev = -1, g_dev_ctxs = 0;

static void claim_device(int device) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (g_dev_ctxs > 0 && g_dev != device)
        fail(CHEBFD_ERR_UNSUPPORTED, "one CUDA device per process: contexts already exist on device " +
                                         std::to_string(g_dev));
    g_dev = device;
    ++g_dev_ctxs;
}

static void release_device() {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (g_dev_ctxs > 0 && --g_dev_ctxs == 0) g_dev = -1;
}

static void ctx_init(Context& c, int device) {
    c.device = device;
    CFD_CUDA(cudaSetDevice(device));
    CFD_CUDA(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, device));
    int l2 = 0;
    CFD_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device));
    if (l2 > 0) c.l2_bytes = l2;
    CFD_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    CFD_CUDA(cudaStreamCreateWithFlags(&c.comm_stream, cudaStreamNonBlocking));
    CFD_CUDA(cudaEventCreateWithFlags(&c.ev_a, cudaEventDisableTiming));
    CFD_CUDA(cudaEventCreateWithFlags(&c.ev_b, cudaEventDisableTiming));
    cublasHandle_t h;
    cublas_check(cublasCreate(&h), "cublasCreate");
    c.cublas = reinterpret_cast<cublasContext*>(h);
    cublas_check(cublasSetStream(h, c.stream), "cublasSetStream");
    // reduction scratch sized for the largest persistent grid (no allocation
    // inside graph capture): grid <= 8 CTAs/SM, up to 3 launches per step,
    // 2 dots x 256 units x 16 B
    c.partials.ensure(static_cast<size_t>(c.num_sms) * 8 * 3 * 2 * 256 * 16);
    c.counter.ensure(4096);  // grid ticket + group tickets of grid_reduce
    CFD_CUDA(cudaMemsetAsync(c.counter.p, 0, 4096, c.stream));
    c.dscratch.ensure(1 << 20);
    // test hook: CHEBFD_GROUPED=2 runs the whole suite on the row-group kernel
    if (const char* e = std::getenv("CHEBFD_GROUPED")) c.grouped = std::atoi(e);
    if (const char* e = std::getenv("CHEBFD_GROUP_LINES")) c.group_lines = std::atoi(e);
    if (const char* e = std::getenv("CHEBFD_RING")) c.ring = std::atoi(e);
    ctx_sync(c);
}

}  // extern "C"

namespace cfd {
// contexts of a virtual rank group (vgroup.cu): same device, no NCCL communicator
Context* create_group_context(int device, int rank, int nranks) {
    claim_device(device);
    try {
        auto c = std::make_unique<Context>();
        ctx_init(*c, device);
        c->rank = rank;
        c->nranks = nranks;
        return c.release();
    } catch (...) {
        release_device();
        throw;
    }
}

void destroy_group_context(Context* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    delete c;
    release_device();
}

}  // namespace cfd

extern "C" {

int chebfd_ctx_create(int device, chebfd_ctx** out) {
    return guard([&] {
        claim_device(device);
        try {
            auto c = std::make_unique<Context>();
            ctx_init(*c, device);
            *out = reinterpret_cast<chebfd_ctx*>(c.release());
        } catch (...) {
            release_device();
            throw;
        }
    });
}

int chebfd_ctx_create_dist(int device, int rank, int nranks, const unsigned char id[128],
                           chebfd_ctx** out) {
    return guard([&] {
        require(nranks >= 1 && rank >= 0 && rank < nranks, "ctx_create_dist: bad rank/nranks");
        claim_device(device);
        try {
            auto c = std::make_unique<Context>();
            ctx_init(*c, device);
            c->rank = rank;
            c->nranks = nranks;
            if (nranks > 1) {
                ncclUniqueId u;
                std::memcpy(u.internal, id, 128);
                nccl_check(ncclCommInitRank(&c->nccl, nranks, u, rank), "ncclCommInitRank");
            }
            *out = reinterpret_cast<chebfd_ctx*>(c.release());
        } catch (...) {
            release_device();
            throw;
        }
    });
}

int chebfd_ctx_destroy(chebfd_ctx* ctx) {
    return guard([&] {
        Context* c = reinterpret_cast<Context*>(ctx);
        if (!c) return;
        cudaSetDevice(c->device);
        delete c;
        release_device();
    });
}

int chebfd_ctx_synchronize(chebfd_ctx* ctx) {
    return guard([&] { ctx_sync(*reinterpret_cast<Context*>(ctx)); });
}

int chebfd_ctx_stream(chebfd_ctx* ctx, void** stream) {
    return guard([&] { *stream = reinterpret_cast<Context*>(ctx)->stream; });
}

int chebfd_ctx_info(chebfd_ctx* ctx, int* device, int* rank, int* nranks, int* num_sms) {
    return guard([&] {
        Context* c = reinterpret_cast<Context*>(ctx);
        if (device) *device = c->device;
        if (rank) *rank = c->rank;
        if (nranks) *nranks = c->nranks;
        if (num_sms) *num_sms = c->num_sms;
    });
}

int chebfd_ctx_launch_count(chebfd_ctx* ctx, int64_t* count) {
    return guard([&] { *count = reinterpret_cast<Context*>(ctx)->launches; });
}

int chebfd_ctx_group_launches(chebfd_ctx* ctx, int64_t* count) {
    return guard([&] { *count = reinterpret_cast<Context*>(ctx)->group_launches; });
}

int chebfd_ctx_ring_launches(chebfd_ctx* ctx, int64_t* count) {
    return guard([&] { *count = reinterpret_cast<Context*>(ctx)->ring_launches; });
}

int chebfd_ctx_band_launches(chebfd_ctx* ctx, int64_t* count) {
    return guard([&] { *count = reinterpret_cast<Context*>(ctx)->band_launches; });
}

int chebfd_ctx_set_option(chebfd_ctx* ctx, int option, int64_t value) {
    return guard([&] {
        Context* c = reinterpret_cast<Context*>(ctx);
        // captured filters bake in the kernel choices: drop them all
        ctx_sync(*c);
        for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second.exec);
        c->graphs.clear();
        if (option == CHEBFD_OPT_GRAPHS)
            c->use_graphs = value != 0;
        else if (option == CHEBFD_OPT_OVERLAP)
            c->overlap = value != 0;
        else if (option == CHEBFD_OPT_KERNEL) {
            if (value == 2 && !CFD_EXPERIMENTAL)
                fail(CHEBFD_ERR_UNSUPPORTED, "kernel variant 2 (staged gathers) needs an EXPERIMENTAL=1 build");
            c->kernel_variant = static_cast<int>(value);
        }
        else if (option == CHEBFD_OPT_SLAB_UNITS)
            c->slab_units = static_cast<int>(value);
        else if (option == CHEBFD_OPT_PAIR) {
            if (value != 0 && !CFD_EXPERIMENTAL)
                fail(CHEBFD_ERR_UNSUPPORTED, "the pair kernel needs an EXPERIMENTAL=1 build");
            c->pair_mode = static_cast<int>(value);
        }
        else if (option == CHEBFD_OPT_MOMENTS)
            c->moments_mode = static_cast<int>(value);
        else if (option == CHEBFD_OPT_PDL)
            c->pdl = static_cast<int>(value);
        else if (option == CHEBFD_OPT_DELAYED_X)
            c->delayed_x = static_cast<int>(value);
        else if (option == CHEBFD_OPT_BAND_BYTES)
            c->band_bytes = value;
        else if (option == CHEBFD_OPT_ASYNC_START)
            c->async_start_entries = value;
        else if (option == CHEBFD_OPT_GRAM)
            c->gram_mode = static_cast<int>(value);
        else if (option == CHEBFD_OPT_COMPACT_HALO)
            c->compact_halo = value != 0;
        else if (option == CHEBFD_OPT_GROUPED)
            c->grouped = static_cast<int>(value);
        else if (option == CHEBFD_OPT_GROUP_LINES)
            c->group_lines = static_cast<int>(value);
        else if (option == CHEBFD_OPT_RING)
            c->ring = static_cast<int>(value);
        else if (option == CHEBFD_OPT_RING_SEGX)
            c->ring_segx = static_cast<int>(value);
        else if (option == CHEBFD_OPT_RING_NO)
            c->ring_no = static_cast<int>(value);
        else if (option == CHEBFD_OPT_RING_NZ)
            c->ring_nz = static_cast<int>(value);
        else if (option == CHEBFD_OPT_RING_ROWS)
            c->ring_rows = static_cast<int>(value);
        else if (option == CHEBFD_OPT_RING_CONSTS)
            c->ring_consts = static_cast<int>(value);
        else if (option == CHEBFD_OPT_RING_TMAP)
            c->ring_tmap = static_cast<int>(value);
        else if (option == CHEBFD_OPT_RING_ORDER)
            c->ring_order = static_cast<int>(value);
        else if (option == CHEBFD_OPT_RING_UNIT)
            c->ring_spb_ctas = static_cast<int>(value);
        else if (option == CHEBFD_OPT_RING_DOTS)
            c->ring_dots = static_cast<int>(value);
        else if (option == CHEBFD_OPT_TILES_PER_CTA)
            c->tiles_per_cta = static_cast<int>(std::max<int64_t>(value, 0));
        else if (option == CHEBFD_OPT_PAIR_TILE_ROWS)
            c->pair_tile_rows = static_cast<int>(value);
        else if (option == CHEBFD_OPT_PAIR_THREADS)
            c->pair_threads = static_cast<int>(value);
        else if (option == CHEBFD_OPT_PAIR_EXTRA)
            c->pair_extra = static_cast<int>(value);
        else if (option == CHEBFD_OPT_PAIR_HINTS)
            c->pair_hints = static_cast<int>(value);
        else if (option == CHEBFD_OPT_PAIR_SLAB)
            c->pair_slab = static_cast<int>(value);
        else
            fail(CHEBFD_ERR_INVALID_ARGUMENT, "unknown option");
    });
}

int chebfd_ctx_event_record(chebfd_ctx* ctx, int slot) {
    return guard([&] {
        Context* c = reinterpret_cast<Context*>(ctx);
        require(slot >= 0 && slot < 16, "event slot out of range");
        if (!c->timers[slot]) CFD_CUDA(cudaEventCreate(&c->timers[slot]));
        CFD_CUDA(cudaEventRecord(c->timers[slot], c->stream));
    });
}

int chebfd_ctx_event_elapsed(chebfd_ctx* ctx, int a, int b, float* ms) {
    return guard([&] {
        Context* c = reinterpret_cast<Context*>(ctx);
        require(a >= 0 && a < 16 && b >= 0 && b < 16 && c->timers[a] && c->timers[b],
                "event slot not recorded");
        CFD_CUDA(cudaEventSynchronize(c->timers[b]));
        CFD_CUDA(cudaEventElapsedTime(ms, c->timers[a], c->timers[b]));
    });
}

int chebfd_host_alloc(size_t bytes, void** out) {
    return guard([&] { CFD_CUDA(cudaMallocHost(out, std::max<size_t>(bytes, 1))); });
}

int chebfd_host_free(void* p) {
    return guard([&] {
        if (p) CFD_CUDA(cudaFreeHost(p));
    });
}

// ---- host CSR generators --------------------------------------------------
static int csr_gen(bool ti, const chebfd_lattice* spec, int64_t r0, int64_t r1, int64_t* dim,
                   int64_t* nnz, int64_t* offs, int64_t* cols, void* vals) {
    return guard([&] {
        require(spec != nullptr, "null lattice spec");
        HostCsr h = ti ? gen_topological_insulator(*spec, r0, r1) : gen_graphene(*spec, r0, r1);
        if (dim) *dim = h.dim;
        *nnz = static_cast<int64_t>(h.cols.size());
        if (offs) {
            std::memcpy(offs, h.offs.data(), sizeof(int64_t) * h.offs.size());
            std::memcpy(cols, h.cols.data(), sizeof(int64_t) * h.cols.size());
            std::memcpy(vals, h.vals.data(), sizeof(double) * h.vals.size());
        }
    });
}

int chebfd_csr_graphene(const chebfd_lattice* spec, int64_t r0, int64_t r1, int64_t* dim,
                        int64_t* nnz, int64_t* offs, int64_t* cols, void* vals) {
    return csr_gen(false, spec, r0, r1, dim, nnz, offs, cols, vals);
}

int chebfd_csr_topological_insulator(const chebfd_lattice* spec, int64_t r0, int64_t r1,
                                     int64_t* dim, int64_t* nnz, int64_t* offs, int64_t* cols,
                                     void* vals) {
    return csr_gen(true, spec, r0, r1, dim, nnz, offs, cols, vals);
}

// ---- matrices ---------------------------------------------------------------
int chebfd_matrix_from_csr(chebfd_ctx* ctx, int kind, int64_t dim, const int64_t* offs,
                           const int64_t* cols, const void* vals, chebfd_matrix** out) {
    return guard([&] {
        Context& c = *reinterpret_cast<Context*>(ctx);
        require(kind == CHEBFD_REAL64 || kind == CHEBFD_COMPLEX128, "bad scalar kind");
        // SparseMatrix::validate (sparse_matrix.hpp:87-100)
        if (dim < 0) fail(CHEBFD_ERR_INVALID_ARGUMENT, "SparseMatrix: negative dimension");
        require(offs != nullptr, "SparseMatrix: row_offsets length must be dim+1");
        const int64_t nnz = offs[dim];
        if (offs[0] != 0 || nnz < 0)
            fail(CHEBFD_ERR_INVALID_ARGUMENT, "SparseMatrix: invalid row_offsets range");
        for (int64_t i = 0; i < dim; ++i)
            if (offs[i] > offs[i + 1])
                fail(CHEBFD_ERR_INVALID_ARGUMENT, "SparseMatrix: row_offsets not monotone");
        for (int64_t p = 0; p < nnz; ++p)
            if (cols[p] < 0 || cols[p] >= dim)
                fail(CHEBFD_ERR_INVALID_ARGUMENT, "SparseMatrix: column index out of range");
        std::vector<int64_t> starts(c.nranks + 1);
        for (int q = 0; q <= c.nranks; ++q) starts[q] = dim * q / c.nranks;
        const int64_t r0 = starts[c.rank], r1 = starts[c.rank + 1];
        HostCsr h;
        h.kind = kind;
        h.dim = dim;
        h.row_begin = r0;
        h.rows = r1 - r0;
        h.offs.resize(h.rows + 1);
        for (int64_t i = 0; i <= h.rows; ++i) h.offs[i] = offs[r0 + i] - offs[r0];
        h.cols.assign(cols + offs[r0], cols + offs[r1]);
        const int f = kind ? 2 : 1;
        const double* v = static_cast<const double*>(vals);
        h.vals.assign(v + f * offs[r0], v + f * offs[r1]);
        const bool herm = csr_is_hermitian(kind, dim, offs, cols, v);
        auto m = matrix_from_host_csr(c, h, r0, r1, starts, nnz, herm);
        m->hermitian = herm;
        *out = reinterpret_cast<chebfd_matrix*>(m.release());
    });
}

int chebfd_matrix_graphene(chebfd_ctx* ctx, const chebfd_lattice* spec, chebfd_matrix** out) {
    return guard([&] {
        require(spec != nullptr, "null lattice spec");
        auto m = lattice_matrix(*reinterpret_cast<Context*>(ctx), *spec, false);
        *out = reinterpret_cast<chebfd_matrix*>(m.release());
    });
}

int chebfd_matrix_topological_insulator(chebfd_ctx* ctx, const chebfd_lattice* spec,
                                        chebfd_matrix** out) {
    return guard([&] {
        require(spec != nullptr, "null lattice spec");
        auto m = lattice_matrix(*reinterpret_cast<Context*>(ctx), *spec, true);
        *out = reinterpret_cast<chebfd_matrix*>(m.release());
    });
}

int chebfd_matrix_destroy(chebfd_matrix* a) {
    return guard([&] {
        Matrix* m = reinterpret_cast<Matrix*>(a);
        if (!m) return;
        ctx_sync(*m->ctx);
        purge_graphs(*m->ctx, m, nullptr);
        delete m;
    });
}

int chebfd_matrix_get_info(const chebfd_matrix* a, chebfd_matrix_info* out) {
    return guard([&] {
        const Matrix* m = reinterpret_cast<const Matrix*>(a);
        out->kind = m->kind;
        out->dim = m->part.dim;
        out->nnz = m->nnz_global;
        out->local_rows = m->part.local;
        out->row_begin = m->part.row_begin;
        out->local_nnz = m->nnz_local;
        out->sell_entries = m->entries;
        out->halo_lo = m->part.halo_lo;
        out->halo_hi = m->part.halo_hi;
        out->chunk = kChunk;
        out->max_row_len = m->max_row_len;
        out->stage_rows = m->stage_max_rows;
    });
}

// ---- blocks -------------------------------------------------------------------
int chebfd_block_create(chebfd_matrix* a, int64_t width, chebfd_block** out) {
    return guard([&] {
        Matrix* m = reinterpret_cast<Matrix*>(a);
        auto b = make_block(*m->ctx, m, m->kind, m->part.local, width);
        *out = reinterpret_cast<chebfd_block*>(b.release());
    });
}

int chebfd_block_create_dim(chebfd_ctx* ctx, int kind, int64_t dim, int64_t width,
                            chebfd_block** out) {
    return guard([&] {
        Context& c = *reinterpret_cast<Context*>(ctx);
        require(kind == CHEBFD_REAL64 || kind == CHEBFD_COMPLEX128, "bad scalar kind");
        auto b = make_block(c, nullptr, kind, dim, width);
        *out = reinterpret_cast<chebfd_block*>(b.release());
    });
}

int chebfd_block_create_like(const chebfd_block* like, int64_t width, chebfd_block** out) {
    return guard([&] {
        require(like != nullptr && out != nullptr, "block_create_like: null argument");
        const Block& l = *reinterpret_cast<const Block*>(like);
        std::unique_ptr<Block> b;
        if (l.shape_of)
            b = make_block(*l.ctx, l.shape_of, l.kind, l.rows, width);
        else
            b = make_block(*l.ctx, nullptr, l.kind, l.rows, width);
        *out = reinterpret_cast<chebfd_block*>(b.release());
    });
}

int chebfd_block_destroy(chebfd_block* b) {
    return guard([&] {
        Block* x = reinterpret_cast<Block*>(b);
        if (!x) return;
        ctx_sync(*x->ctx);
        purge_graphs(*x->ctx, nullptr, x->owned());
        delete x;
    });
}

int chebfd_block_info(const chebfd_block* b, int* kind, int64_t* rows, int64_t* width,
                      int64_t* row_begin) {
    return guard([&] {
        const Block* x = reinterpret_cast<const Block*>(b);
        if (kind) *kind = x->kind;
        if (rows) *rows = x->rows;
        if (width) *width = x->width;
        if (row_begin) *row_begin = x->row_begin;
    });
}

int chebfd_block_upload(chebfd_block* b, const void* host) {
    return guard([&] {
        Block* x = reinterpret_cast<Block*>(b);
        if (x->owned_bytes())
            CFD_CUDA(cudaMemcpyAsync(x->owned(), host, x->owned_bytes(), cudaMemcpyHostToDevice,
                                     x->ctx->stream));
        ctx_sync(*x->ctx);
    });
}

int chebfd_block_download(const chebfd_block* b, void* host) {
    return guard([&] {
        const Block* x = reinterpret_cast<const Block*>(b);
        if (x->owned_bytes())
            CFD_CUDA(cudaMemcpyAsync(host, x->owned(), x->owned_bytes(), cudaMemcpyDeviceToHost,
                                     x->ctx->stream));
        ctx_sync(*x->ctx);
    });
}

int chebfd_block_copy(chebfd_block* dst, const chebfd_block* src) {
    return guard([&] {
        Block* d = reinterpret_cast<Block*>(dst);
        const Block* s = reinterpret_cast<const Block*>(src);
        check_same_shape(*d, *s);
        if (d->owned_bytes())
            CFD_CUDA(cudaMemcpyAsync(d->owned(), s->owned(), d->owned_bytes(),
                                     cudaMemcpyDeviceToDevice, d->ctx->stream));
    });
}

int chebfd_block_zero(chebfd_block* b) {
    return guard([&] {
        Block* x = reinterpret_cast<Block*>(b);
        CFD_CUDA(cudaMemsetAsync(x->buf.p, 0, x->buf.bytes, x->ctx->stream));
    });
}

int chebfd_block_randomize(chebfd_block* b, uint64_t seed) {
    return guard([&] { randomize_upload(*reinterpret_cast<Block*>(b)->ctx, *reinterpret_cast<Block*>(b), seed); });
}

int chebfd_block_randomize_device(chebfd_block* b, uint64_t seed) {
    return guard([&] {
        Block* x = reinterpret_cast<Block*>(b);
        launch_philox_normal(*x->ctx, *x, seed, x->ctx->stream);
    });
}

int chebfd_block_scale_columns(chebfd_block* b, const double* s) {
    // x(:,k) /= d[k] semantics are used internally; the public entry point
    // multiplies, so pass reciprocals to the divide kernel exactly: store d = 1/s
    return guard([&] {
        Block* x = reinterpret_cast<Block*>(b);
        Context& c = *x->ctx;
        std::vector<double> d(static_cast<size_t>(x->width));
        for (int64_t k = 0; k < x->width; ++k) d[k] = 1.0 / s[k];
        c.dscratch.ensure(sizeof(double) * d.size());
        CFD_CUDA(cudaMemcpyAsync(c.dscratch.p, d.data(), sizeof(double) * d.size(),
                                 cudaMemcpyHostToDevice, c.stream));
        launch_scale_columns(c, *x, c.dscratch.as<double>(), c.stream);
        ctx_sync(c);
    });
}

int chebfd_block_copy_columns(chebfd_block* dst, int64_t d0, const chebfd_block* src, int64_t s0,
                              int64_t n) {
    return guard([&] {
        Block* d = reinterpret_cast<Block*>(dst);
        const Block* s = reinterpret_cast<const Block*>(src);
        require(d->rows == s->rows && d->kind == s->kind, "copy_columns: shape mismatch");
        require(d0 >= 0 && s0 >= 0 && n >= 0 && d0 + n <= d->width && s0 + n <= s->width,
                "copy_columns: column range out of bounds");
        launch_copy_columns(*d->ctx, *d, d0, *s, s0, n, d->ctx->stream);
    });
}

int chebfd_block_device_ptr(chebfd_block* b, void** ptr) {
    return guard([&] { *ptr = reinterpret_cast<Block*>(b)->owned(); });
}

// ---- kernels ----------------------------------------------------------------------
int chebfd_spmmvm(chebfd_matrix* a, chebfd_block* x, chebfd_block* y, double alpha, double beta) {
    return guard([&] {
        Matrix& m = *reinterpret_cast<Matrix*>(a);
        Block& X = *reinterpret_cast<Block*>(x);
        Block& Y = *reinterpret_cast<Block*>(y);
        check_conforms(m, X, "spmmvm");
        check_same_shape(X, Y);
        require(X.owned() != Y.owned(), "spmmvm: X and Y must not alias");
        StepArgs s{};
        s.kind_step = kStepSpmmvm;
        s.w = Y.owned();
        s.alpha = alpha;
        s.beta = beta;
        run_step_all(*m.ctx, m, s, X);
    });
}

int chebfd_spmmvm_fused(chebfd_matrix* a, chebfd_block* u, chebfd_block* w, chebfd_block* x,
                        double alpha, double beta, double coeff, void* dots) {
    return guard([&] {
        Matrix& m = *reinterpret_cast<Matrix*>(a);
        Block& U = *reinterpret_cast<Block*>(u);
        Block& W = *reinterpret_cast<Block*>(w);
        Block& X = *reinterpret_cast<Block*>(x);
        check_same_shape(U, W);  // kernels.hpp:77-81
        check_same_shape(U, X);
        check_conforms(m, U, "spmmvm_fused");
        if (U.owned() == W.owned() || U.owned() == X.owned() || W.owned() == X.owned())
            fail(CHEBFD_ERR_INVALID_ARGUMENT, "spmmvm_fused: U, W, X must not alias");
        Context& c = *m.ctx;
        StepArgs s{};
        s.kind_step = kStepFused;
        s.w = W.owned();
        s.x = X.owned();
        s.alpha = 2.0 * alpha;
        s.beta = 2.0 * beta;
        s.c0 = coeff;
        s.dots_mode = dots ? 1 : 0;
        const size_t bytes = static_cast<size_t>(U.width) * U.scalar_bytes();
        if (dots) {
            c.dscratch.ensure(bytes);
            s.dots_out = c.dscratch.p;
        }
        run_step_all(c, m, s, U);
        if (dots) {
            allreduce_sum(c, c.dscratch.as<double>(), bytes / 8, c.stream);
            CFD_CUDA(cudaMemcpyAsync(dots, c.dscratch.p, bytes, cudaMemcpyDeviceToHost, c.stream));
            ctx_sync(c);
        }
    });
}

int chebfd_recurrence_step(chebfd_matrix* a, chebfd_block* u, chebfd_block* w, double alpha,
                           double beta) {
    return guard([&] {
        Matrix& m = *reinterpret_cast<Matrix*>(a);
        Block& U = *reinterpret_cast<Block*>(u);
        Block& W = *reinterpret_cast<Block*>(w);
        check_same_shape(U, W);
        check_conforms(m, U, "recurrence_step");
        if (U.owned() == W.owned())
            fail(CHEBFD_ERR_INVALID_ARGUMENT, "recurrence_step: U and W must not alias");
        StepArgs s{};
        s.kind_step = kStepRecur;
        s.w = W.owned();
        s.alpha = 2.0 * alpha;
        s.beta = 2.0 * beta;
        run_step_all(*m.ctx, m, s, U);
    });
}

int chebfd_block_axpy_scal(chebfd_block* x, const chebfd_block* u, const chebfd_block* w,
                           double c0, double c1, double c2) {
    return guard([&] {
        Block& X = *reinterpret_cast<Block*>(x);
        const Block& U = *reinterpret_cast<const Block*>(u);
        const Block& W = *reinterpret_cast<const Block*>(w);
        check_same_shape(X, U);
        check_same_shape(X, W);
        launch_axpy(*X.ctx, X, U, W, c0, c1, c2, X.ctx->stream);
    });
}

int chebfd_column_dots(const chebfd_block* x, const chebfd_block* y, void* out) {
    return guard([&] {
        const Block& X = *reinterpret_cast<const Block*>(x);
        column_dots_host(*X.ctx, X, *reinterpret_cast<const Block*>(y), out);
    });
}

int chebfd_column_norms(const chebfd_block* x, double* out) {
    return guard([&] {
        const Block& X = *reinterpret_cast<const Block*>(x);
        std::vector<double> d(static_cast<size_t>(X.width) * (X.kind ? 2 : 1));
        column_dots_host(*X.ctx, X, X, d.data());
        for (int64_t k = 0; k < X.width; ++k) out[k] = std::sqrt(X.kind ? d[2 * k] : d[k]);
    });
}

int chebfd_gram(const chebfd_block* x, const chebfd_block* y, void* out) {
    return guard([&] {
        const Block& X = *reinterpret_cast<const Block*>(x);
        gram_host(*X.ctx, X, *reinterpret_cast<const Block*>(y), out);
    });
}

int chebfd_block_mult_small(const chebfd_block* x, const void* b, int64_t bcols, chebfd_block* y) {
    return guard([&] {
        const Block& X = *reinterpret_cast<const Block*>(x);
        Block& Y = *reinterpret_cast<Block*>(y);
        require(Y.rows == X.rows && Y.kind == X.kind && Y.width == bcols,
                "block_mult_small: shape mismatch");
        require(X.owned() != Y.owned(), "block_mult_small: X and Y must not alias");
        mult_small_host_b(*X.ctx, X, b, bcols, Y);
    });
}

// ---- filter ------------------------------------------------------------------------
int chebfd_window_coeffs(double tlo, double thi, double blo, double bhi, int degree, double* out) {
    return guard([&] {
        auto c = window_coeffs(tlo, thi, blo, bhi, degree);
        std::memcpy(out, c.data(), sizeof(double) * c.size());
    });
}

int chebfd_kernel_coeffs(int kernel, int mu, int degree, double* out) {
    return guard([&] {
        auto g = kernel_coeffs(kernel, mu, degree);
        std::memcpy(out, g.data(), sizeof(double) * g.size());
    });
}

int chebfd_make_filter(double tlo, double thi, double blo, double bhi, int degree, int kernel,
                       int mu, double* combined, double* alpha, double* beta) {
    return guard([&] {
        // make_filter (filter.cpp:86-99)
        auto c = window_coeffs(tlo, thi, blo, bhi, degree);
        auto g = kernel_coeffs(kernel, mu, degree);
        for (size_t n = 0; n < c.size(); ++n) combined[n] = g[n] * c[n];
        *alpha = 2.0 / (bhi - blo);
        *beta = (blo + bhi) / (blo - bhi);
    });
}

int chebfd_eval_scalar(const double* combined, int degree, double alpha, double beta, double blo,
                       double bhi, double x, double* out) {
    return guard([&] {
        // eval_scalar (filter.cpp:101-114)
        if (x < blo || x > bhi)
            fail(CHEBFD_ERR_DOMAIN, "eval_scalar: x outside expansion bounds");
        const double t = alpha * x + beta;
        double tm2 = 1.0, tm1 = t;
        double acc = combined[0] + combined[1] * t;
        for (int n = 2; n <= degree; ++n) {
            const double tn = 2.0 * t * tm1 - tm2;
            acc += combined[n] * tn;
            tm2 = tm1;
            tm1 = tn;
        }
        *out = acc;
    });
}

int chebfd_apply_filter(chebfd_matrix* a, chebfd_block* x, const double* combined, int degree,
                        double alpha, double beta, double* moments) {
    return guard([&] {
        Matrix& m = *reinterpret_cast<Matrix*>(a);
        apply_filter_device(*m.ctx, m, *reinterpret_cast<Block*>(x), combined, degree, alpha, beta,
                            moments);
    });
}

int chebfd_apply_filter_host(chebfd_matrix* a, void* x_host, int64_t width, const double* combined,
                             int degree, double alpha, double beta, double* moments) {
    return guard([&] {
        Matrix& m = *reinterpret_cast<Matrix*>(a);
        Context& c = *m.ctx;
        if (degree < 2) fail(CHEBFD_ERR_INVALID_ARGUMENT, "apply_filter: degree must be >= 2");
        // a cached device block per (matrix, width) receives the host data
        auto key = std::make_tuple(static_cast<const void*>(&m), width, -1 - m.kind);
        FilterWorkspace& io = c.filter_ws[key];
        if (!io.u) io.u = make_block(c, &m, m.kind, m.part.local, width);
        Block& X = *io.u;
        CFD_CUDA(cudaMemcpyAsync(X.owned(), x_host, X.owned_bytes(), cudaMemcpyHostToDevice,
                                 c.stream));
        apply_filter_device(c, m, X, combined, degree, alpha, beta, moments);
        CFD_CUDA(cudaMemcpyAsync(x_host, X.owned(), X.owned_bytes(), cudaMemcpyDeviceToHost,
                                 c.stream));
        ctx_sync(c);
    });
}

// ---- streamed host filtering ------------------------------------------------------
struct FilterPipe {
    Context* c = nullptr;
    Matrix* m = nullptr;
    int64_t width = 0;
    std::unique_ptr<Block> slot[2];
    DeviceBuffer gram[2];  // per-slot device Gram of the filtered block (submit_gram)
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t in_ready[2] = {}, done[2] = {}, out_done[2] = {};
    bool used[2] = {false, false};
    int next = 0;
    ~FilterPipe() {
        if (h2d) cudaStreamSynchronize(h2d);
        if (d2h) cudaStreamSynchronize(d2h);
        if (c) cudaStreamSynchronize(c->stream);
        for (int i = 0; i < 2; ++i) {
            if (in_ready[i]) cudaEventDestroy(in_ready[i]);
            if (done[i]) cudaEventDestroy(done[i]);
            if (out_done[i]) cudaEventDestroy(out_done[i]);
        }
        if (h2d) cudaStreamDestroy(h2d);
        if (d2h) cudaStreamDestroy(d2h);
    }
};

int chebfd_filter_pipe_create(chebfd_matrix* a, int64_t width, chebfd_filter_pipe** out) {
    return guard([&] {
        require(a != nullptr && out != nullptr, "filter_pipe_create: null argument");
        require(width >= 1, "filter_pipe_create: width must be >= 1");
        Matrix& m = *reinterpret_cast<Matrix*>(a);
        auto p = std::make_unique<FilterPipe>();
        p->c = m.ctx;
        p->m = &m;
        p->width = width;
        for (int i = 0; i < 2; ++i) {
            p->slot[i] = make_block(*m.ctx, &m, m.kind, m.part.local, width);
            CFD_CUDA(cudaEventCreateWithFlags(&p->in_ready[i], cudaEventDisableTiming));
            CFD_CUDA(cudaEventCreateWithFlags(&p->done[i], cudaEventDisableTiming));
            CFD_CUDA(cudaEventCreateWithFlags(&p->out_done[i], cudaEventDisableTiming));
        }
        CFD_CUDA(cudaStreamCreateWithFlags(&p->h2d, cudaStreamNonBlocking));
        CFD_CUDA(cudaStreamCreateWithFlags(&p->d2h, cudaStreamNonBlocking));
        *out = reinterpret_cast<chebfd_filter_pipe*>(p.release());
    });
}

static void pipe_submit(FilterPipe& p, const void* host_in, void* host_out, const double* combined,
                        int degree, double alpha, double beta, void* gram_host);

int chebfd_filter_pipe_submit(chebfd_filter_pipe* pipe, const void* host_in, void* host_out,
                              const double* combined, int degree, double alpha, double beta) {
    return guard([&] {
        require(pipe != nullptr && host_in != nullptr && host_out != nullptr,
                "filter_pipe_submit: null argument");
        pipe_submit(*reinterpret_cast<FilterPipe*>(pipe), host_in, host_out, combined, degree, alpha,
                    beta, nullptr);
    });
}

int chebfd_filter_pipe_submit_gram(chebfd_filter_pipe* pipe, const void* host_in, void* host_out,
                                   const double* combined, int degree, double alpha, double beta,
                                   void* gram_host) {
    return guard([&] {
        require(pipe != nullptr && host_in != nullptr && host_out != nullptr && gram_host != nullptr,
                "filter_pipe_submit_gram: null argument");
        pipe_submit(*reinterpret_cast<FilterPipe*>(pipe), host_in, host_out, combined, degree, alpha,
                    beta, gram_host);
    });
}

static void pipe_submit(FilterPipe& p, const void* host_in, void* host_out, const double* combined,
                        int degree, double alpha, double beta, void* gram_host) {
    {
        if (degree < 2) fail(CHEBFD_ERR_INVALID_ARGUMENT, "apply_filter: degree must be >= 2");
        Context& c = *p.c;
        const int s = p.next;
        p.next ^= 1;
        Block& X = *p.slot[s];
        // the slot's previous result must have left before new input lands in it
        if (p.used[s]) CFD_CUDA(cudaStreamWaitEvent(p.h2d, p.out_done[s], 0));
        CFD_CUDA(cudaMemcpyAsync(X.owned(), host_in, X.owned_bytes(), cudaMemcpyHostToDevice, p.h2d));
        CFD_CUDA(cudaEventRecord(p.in_ready[s], p.h2d));
        CFD_CUDA(cudaStreamWaitEvent(c.stream, p.in_ready[s], 0));
        apply_filter_device(c, *p.m, X, combined, degree, alpha, beta, nullptr);
        const size_t gbytes = static_cast<size_t>(X.width * X.width) * X.scalar_bytes();
        if (gram_host) {
            // the Rayleigh-Ritz Gram X^H X of the filtered block (kernels.hpp:165-192),
            // all-reduced over ranks, into the slot's device buffer
            p.gram[s].ensure(gbytes);
            gemm_gram(c, X, X, p.gram[s].p);
            allreduce_sum(c, p.gram[s].as<double>(), gbytes / 8, c.stream);
        }
        CFD_CUDA(cudaEventRecord(p.done[s], c.stream));
        CFD_CUDA(cudaStreamWaitEvent(p.d2h, p.done[s], 0));
        CFD_CUDA(cudaMemcpyAsync(host_out, X.owned(), X.owned_bytes(), cudaMemcpyDeviceToHost, p.d2h));
        if (gram_host)
            CFD_CUDA(cudaMemcpyAsync(gram_host, p.gram[s].p, gbytes, cudaMemcpyDeviceToHost, p.d2h));
        CFD_CUDA(cudaEventRecord(p.out_done[s], p.d2h));
        p.used[s] = true;
    }
}

int chebfd_filter_pipe_wait(chebfd_filter_pipe* pipe) {
    return guard([&] {
        require(pipe != nullptr, "filter_pipe_wait: null pipe");
        FilterPipe& p = *reinterpret_cast<FilterPipe*>(pipe);
        CFD_CUDA(cudaStreamSynchronize(p.d2h));
        CFD_CUDA(cudaStreamSynchronize(p.c->stream));
    });
}

int chebfd_filter_pipe_destroy(chebfd_filter_pipe* pipe) {
    return guard([&] { delete reinterpret_cast<FilterPipe*>(pipe); });
}

}  // extern "C"
