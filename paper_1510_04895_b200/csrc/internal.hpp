// Internal declarations of the chebfd_b200 library (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/chebfd_b200.h"

// Opt-in kernel variants that measured slower than the default path (the two-step
// wavefront pair kernel, pair.cu, and the staged-gather step kernel, kernel variant 2;
// DESIGN.md §5): compiled only with -DCFD_EXPERIMENTAL=1 (make EXPERIMENTAL=1).
#ifndef CFD_EXPERIMENTAL
#define CFD_EXPERIMENTAL 0
#endif

struct cublasContext;
struct cusolverDnContext;
typedef struct ncclComm* ncclComm_t;

namespace cfd {

// ---- errors: internal C++ exceptions mapped to status codes at the ABI --------
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void require(bool ok, const std::string& msg) {
    if (!ok) fail(CHEBFD_ERR_INVALID_ARGUMENT, msg);
}
void cuda_check(cudaError_t e, const char* what);
#define CFD_CUDA(x) ::cfd::cuda_check((x), #x)

// ---- device memory --------------------------------------------------------------
struct DeviceBuffer {
    void* p = nullptr;
    size_t bytes = 0;
    DeviceBuffer() = default;
    explicit DeviceBuffer(size_t n);
    ~DeviceBuffer();
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    void ensure(size_t n);  // grow-only
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

// ---- row partition of a distributed operator ---------------------------------------
// Rows [row_begin, row_begin+local) are owned.  Gathered operands live in an
// extended row space [halo_lo | owned | halo_hi]; halo_lo holds the global
// rows [lo_src_begin, lo_src_begin+halo_lo) owned by rank lo_rank, halo_hi
// the rows [hi_src_begin, ...) owned by hi_rank.
struct Partition {
    int64_t dim = 0;  // global
    int64_t row_begin = 0, local = 0;
    int64_t halo_lo = 0, halo_hi = 0;
    int64_t lo_src_begin = 0, hi_src_begin = 0;
    int lo_rank = -1, hi_rank = -1;
    // rows that read the halo: [0, bnd_lo) and [local - bnd_hi, local)
    int64_t bnd_lo = 0, bnd_hi = 0;
    // neighbours' requests of our rows: we send rows [send_lo_begin, +send_lo_n)
    // (local index) to lo_rank and [send_hi_begin, +send_hi_n) to hi_rank
    int64_t send_lo_begin = 0, send_lo_n = 0, send_hi_begin = 0, send_hi_n = 0;
    int64_t ext_rows() const { return halo_lo + local + halo_hi; }
    // Compact halos (structurally symmetric operators, e.g. the lattice models): only the
    // neighbour rows the local rows actually reference are exchanged -- TI reads orbitals
    // {0,3} of the plane below and {1,2} of the plane above, half of each plane.  The
    // halo regions then hold halo_lo_rows / halo_hi_rows (sorted global rows) in order,
    // and this rank sends its rows send_lo_rows / send_hi_rows (sorted local indices).
    // By structural symmetry a neighbour's halo list equals our send list to it.
    bool compact = false;
    std::vector<int64_t> halo_lo_rows, halo_hi_rows, send_lo_rows, send_hi_rows;
};

// Extended-row index of global column g in a partition (-2: not held).  Used
// by the SELL builder on the device and by the host planning API.
#ifdef __CUDACC__
#define CFD_HD __host__ __device__
#else
#define CFD_HD
#endif
struct ColMap {
    int64_t row_begin, local, halo_lo, halo_hi, lo_src, hi_src;
    CFD_HD int64_t map(int64_t g) const {
        if (g >= row_begin && g < row_begin + local) return g - row_begin + halo_lo;
        if (g >= lo_src && g < lo_src + halo_lo) return g - lo_src;
        if (g >= hi_src && g < hi_src + halo_hi) return g - hi_src + halo_lo + local;
        return -2;
    }
};
inline ColMap colmap_of(const Partition& p) {
    return ColMap{p.row_begin, p.local, p.halo_lo, p.halo_hi, p.lo_src_begin, p.hi_src_begin};
}

struct Context;

// ---- SELL-C-sigma matrix (C = 32, sigma = 1) ---------------------------------------
constexpr int kChunk = 32;
constexpr int kStageRuns = 64;  // row runs per chunk in a staged-gather plan
constexpr int kStageGap = 3;    // runs closer than this many rows are merged (copied together)

// ---- grouped matrix: row groups of 4 with merged (union) column lists ---------------
// Rows 4g .. 4g+3 share one list of gathered columns: entry k = extended-row index
// (low 28 bits) | row mask (high 4 bits); for every set bit r, in increasing r, the next
// value of the group multiplies in[col] into row r's sum.  Each row meets its entries in
// its CSR order (the merge keeps every row's order), so the sums are bit-identical to the
// SELL kernels; a lattice site's 4 orbitals share their 24 neighbour rows instead of
// gathering 44 (TI), which halves the L1 traffic of a step.
// Tiles of kTileGroups groups (64 rows) are contiguous: cols = [int4 header per group:
// (column offset in the tile's segment, value offset, padded column count, column count)]
// + the groups' packed columns (padded to multiples of 4 with mask-0 copies);
// vals = the groups' values in processing order.
constexpr int kGroupRows = 4;
constexpr int kTileGroups = 16;
constexpr int kTileRows = kGroupRows * kTileGroups;
constexpr int kGroupMaxRowLen = 32;  // longer rows: no grouped form
struct GroupedMatrix {
    bool ok = false;
    int64_t ntiles = 0;
    DeviceBuffer tile_cptr;  // int64[ntiles+1]: first int of tile t in cols
    DeviceBuffer tile_vptr;  // int64[ntiles+1]: first value of tile t in vals
    DeviceBuffer cols;       // int32
    DeviceBuffer vals;       // double / double2
    int64_t ncols = 0, nvals = 0;
    int max_tile_cols = 0, max_tile_vals = 0;  // per-tile maxima (shared-memory stage size)
    // Lattice operators: a tile is a patch of il_lines lattice lines x (16 / il_lines)
    // sites instead of 16 consecutive sites, so the y -+ 1 neighbour rows of its groups are
    // each other's own rows and reach the L1 once (il_line_rows rows per line; 0: linear
    // tiles).  Tile t still covers rows inside [64 t', 64 t' + 64)'s line group, so every
    // launch range of whole line groups is the same set of tiles in both numberings.
    int64_t il_line_rows = 0;
    int il_lines = 1;
    std::vector<std::pair<double, std::unique_ptr<DeviceBuffer>>> scaled;
    // Site-ring plan (step_ring.cuh; complex lattice operators with linear tiles): two int4
    // per group -- static-pattern sites: (z-1 row a, z-1 row b, z+1 row a, z+1 row b)
    // extended-row indices or -1; generic sites: (column-list offset lo, hi, padded column
    // count, 0) -- then (value offset lo, hi, pattern id, value count).  ring_ok: every
    // static site's x / y neighbour columns are its lattice neighbours' rows and no site
    // holds more than kRingMaxVals values.
    bool ring_ok = false;
    DeviceBuffer ring_plan;
    // every static site of a pattern holds the same off-diagonal values (the lattice models'
    // hopping terms): ring_consts[pattern id - 1][value index] = that value (unscaled), so
    // the site-ring kernel multiplies with kernel-parameter constants and reads only the
    // four diagonal (disorder) values per site from memory
    bool ring_const_ok = false;
    double ring_consts[3][44][2] = {};
    bool ring_pat_present[3] = {};  // the lattice holds sites of this pattern (else its constants are unset)
};
constexpr int kRingMaxVals = 44;  // values per site staged by the site-ring kernel

struct Matrix {
    Context* ctx = nullptr;
    int kind = 0;
    int64_t nnz_global = 0, nnz_local = 0;
    int max_row_len = 0;
    Partition part;
    int64_t nchunks = 0;
    int64_t entries = 0;     // SELL slots (padding included)
    DeviceBuffer chunk_ptr;  // int64[nchunks+1], slot offsets
    DeviceBuffer chunk_full; // uint8[nchunks]: every row has exactly the chunk width
    // staged-gather plan (kernel variant 2), per 32-row chunk: the rows of the
    // gathered operand the chunk reads, as merged runs copied by TMA into
    // shared memory, and each slot's / own row's index inside that copy
    DeviceBuffer stage_runs;  // int4[nchunks * kStageRuns]: (first ext row, rows, local offset, 0)
    DeviceBuffer stage_meta;  // int2[nchunks]: (runs, rows)
    DeviceBuffer stage_lcol;  // uint16[nchunks * 32 * 16]: row-major within the chunk, 0xFFFF = padding
    DeviceBuffer stage_lown;  // uint16[nchunks * 32]
    int stage_max_rows = 0;   // largest per-chunk row union (0: no plan)
    DeviceBuffer cols;       // int32[entries], extended-row index or -1 padding
    DeviceBuffer vals;       // double or double2 [entries]
    // value copies pre-multiplied by a step's alpha (apply_filter uses alpha
    // and 2 alpha); at most 4 are kept
    std::vector<std::pair<double, std::unique_ptr<DeviceBuffer>>> scaled;
    bool scaled_evicted = false;
    bool hermitian = false; // bitwise A = A^H (lattice models; checked for from_csr input):
                            // enables moment doubling
    int64_t band = 0;       // max |extended column - extended row| over all entries
    // lattice structure of model operators (0: unknown): rows per z-plane and per lattice
    // line (TI: 4 Lx Ly and 4 Lx); the step kernels' band tile order uses it
    int64_t plane_rows = 0, line_rows = 0;
    DeviceBuffer pair_sync; // pair kernel: item / exit tickets + per-1024-row group counters (zeroed)
    // compact halos: this rank's rows sent to lo / hi (local indices, device), the pack
    // buffers they are gathered into before ncclSend, and -- virtual groups -- the
    // neighbours' local indices of this rank's halo rows (pulled by a gather kernel)
    DeviceBuffer send_lo_idx, send_hi_idx, pack_lo, pack_hi, recv_lo_src, recv_hi_src;
    GroupedMatrix grp;  // grouped form (default step kernel where it applies)
};

// ---- block vector -------------------------------------------------------------------
struct Block {
    Context* ctx = nullptr;
    int kind = 0;
    int64_t rows = 0;   // owned rows
    int64_t width = 0;
    int64_t halo_lo = 0, halo_hi = 0;  // extra rows (gather halos)
    int64_t row_begin = 0, dim_global = 0;
    const Matrix* shape_of = nullptr;  // partition the halos belong to (may be null)
    DeviceBuffer buf;   // (halo_lo + rows + halo_hi) x width scalars
    ~Block();           // storage goes back to the context's block cache
    size_t scalar_bytes() const { return kind ? 16 : 8; }
    void* base() const { return buf.p; }  // extended row 0
    void* owned() const {
        return static_cast<char*>(buf.p) + halo_lo * width * scalar_bytes();
    }
    size_t owned_bytes() const { return static_cast<size_t>(rows * width) * scalar_bytes(); }
};

// ---- context -----------------------------------------------------------------------
struct GraphKey {
    const void* a;
    const void* x;
    int degree;
    uint64_t alpha_bits, beta_bits;
    bool moments;
    int64_t width;
    bool operator<(const GraphKey& o) const {
        return std::tie(a, x, degree, alpha_bits, beta_bits, moments, width) <
               std::tie(o.a, o.x, o.degree, o.alpha_bits, o.beta_bits, o.moments, o.width);
    }
};

struct DeviceBuffer;
// A captured apply_filter: the graph reads its coefficients from `coeff`
// (refreshed before every replay) and writes moments into `moments`.
struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    std::shared_ptr<DeviceBuffer> coeff, moments;
    int64_t kernels = 0;
    // the coefficients now in `coeff`: a replay with the same filter skips the host ->
    // device copy (a pageable copy would first wait for the stream to drain, which
    // serialises streamed submissions behind the previous filter)
    std::vector<double> coeff_host;
};

struct FilterWorkspace {
    std::unique_ptr<Block> u, w, x0;
};

struct Context {
    int device = 0, rank = 0, nranks = 1, num_sms = 148;
    double l2_bytes = 126.0 * (1 << 20);
    cudaStream_t stream = nullptr;       // compute
    cudaStream_t comm_stream = nullptr;  // halo exchange
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    cudaEvent_t timers[16] = {};
    cublasContext* cublas = nullptr;
    cusolverDnContext* cusolver = nullptr;
    ncclComm_t nccl = nullptr;
    bool use_graphs = true, overlap = true;
    int kernel_variant = 1;  // step kernel: 0 register gathers, 1 TMA-staged matrix chunks,
                             // 2 TMA-staged matrix chunks + gathered rows (where a plan fits)
    int64_t launches = 0;
    int64_t band_launches = 0;  // step launches that ran in the band (2.5D) tile order
    int slab_units = 0;   // step kernel column-slab width in 16-byte units (0: up to 256)
    // two fused steps per launch (pair.cu): 0 off, 1 where the wavefront's working set
    // fits the L2, 2 wherever the kernel applies; tuning knobs (0 / -1: automatic)
    // filter / KPM moments: 0 direct <x0, T_n x0> per step (x0 stream), 1 doubling from
    // <V_n, V_n>, <V_n, V_n+1> where the operator is Hermitian (default)
    int moments_mode = 1;
    // step kernels of apply_filter / KPM launch as programmatic dependents of the previous
    // step (their set-up overlaps its tail), single-rank operators
    int pdl = 1;  // 0 off, 1 small operators (launch-bound), 2 every single-rank step
    // apply_filter: X read and written every delayed_x-th step (kStepRecur steps, then
    // kStepFusedX2 / X3 adding their terms); 0 or 1: every step
    int delayed_x = 3;
    // band tile order of lattice operators: a band slice of the gathered operand is at
    // most this many bytes (0: row order everywhere); CHEBFD_OPT_BAND_BYTES
    int64_t band_bytes = int64_t(16) << 20;
    // solve with N_S given: blocks of at least this many entries get their start block
    // generated on a helper thread during bounds + KPM (0: never); CHEBFD_OPT_ASYNC_START
    int64_t async_start_entries = int64_t(1) << 26;
    int pair_mode = 0, pair_tile_rows = 0, pair_threads = 0, pair_extra = -1, pair_hints = 1,
        pair_slab = 0;
    // reduction scratch shared by all kernels on `stream` (stream-ordered reuse)
    DeviceBuffer partials;   // per-block partial sums
    DeviceBuffer counter;    // last-block-done ticket (uint32), self-resetting
    // step launches without dots: non-persistent grids of this many consecutive row tiles
    // per CTA (0: persistent CTA-strided grids everywhere); CHEBFD_OPT_TILES_PER_CTA
    int tiles_per_cta = 2;
    // row-group step kernel (step_group.cuh) where the grouped form applies;
    // CHEBFD_OPT_GROUPED (0: SELL kernels only)
    int grouped = 1;
    int group_lines = 1;  // lattice lines per tile of the grouped form (1: linear); set before
                          // building matrices (CHEBFD_OPT_GROUP_LINES)
    int64_t group_launches = 0;  // step launches that ran the row-group kernel
    // site-ring step kernel (step_ring.cuh): 0 off, 1 (default) on lattices whose z-plane of
    // the block exceeds 2 x band_bytes, 2 wherever it applies; CHEBFD_OPT_RING.  ring_segx / ring_no /
    // ring_nz: x-columns per CTA and ring depths (0: defaults); CHEBFD_OPT_RING_SEGX / _NO / _NZ
    int ring = 1, ring_segx = 0, ring_no = 0, ring_nz = 0;
    int ring_order = 3;   // CTA order: 0 x segments fastest (bands of band_bytes), 1 x segments slowest in bands of strips,
                          // 2 planes fastest, then strips, x segments slowest, 3 (default) 2 on shallow slabs else 0;
                          // CHEBFD_OPT_RING_ORDER
    int ring_spb_ctas = 0;  // order 1: CTAs per (segment, band) unit (0: the SM count); CHEBFD_OPT_RING_UNIT
    int ring_tmap = 1;    // tensor-map TMA copies: 1 for column slabs, 2 always, 0 never; CHEBFD_OPT_RING_TMAP
    int ring_consts = 1;  // 1: constant off-diagonal values as kernel parameters where the matrix has them; CHEBFD_OPT_RING_CONSTS
    int ring_dots = 1;  // 1: V_n-only steps with doubling moment sums (DMODE 4 / 5 / 6) on the site-ring kernel; CHEBFD_OPT_RING_DOTS
    int ring_rows = 0;  // rows of a site per consumer thread (4, 2, 1; 0: default 2); CHEBFD_OPT_RING_ROWS
    int64_t ring_launches = 0;   // step launches that ran the site-ring kernel
    // exchange only the referenced halo rows of structurally symmetric operators (lattice
    // models, bitwise-Hermitian from_csr input); CHEBFD_OPT_COMPACT_HALO
    bool compact_halo = true;
    struct VGroup* vgroup = nullptr;  // virtual rank group this context belongs to (vgroup.cu)
    DeviceBuffer dscratch;   // small device results (dots, Gram, moments)
    DeviceBuffer workspace;  // cuSOLVER / misc
    DeviceBuffer devinfo;
    DeviceBuffer coeffs;     // filter coefficients (device copy)
    DeviceBuffer gram_scratch;  // DMMA Gram: split-K partial tiles
    // DMMA Gram super-tile lists per (nx, ny, Hermitian) (uploaded once: no per-call
    // pageable copy, which would wait for the stream to drain)
    std::map<std::tuple<int, int, bool>, std::unique_ptr<DeviceBuffer>> gram_tiles;
    int gram_mode = 1;       // X^H Y: 1 hand-written DMMA kernel (gram.cu), 0 cuBLAS; CHEBFD_OPT_GRAM
    DeviceBuffer small[4];   // host-fed small operands (rotations, eigenvalues, Gram, eig)
    // exact-size cache of block storage: the solver allocates the same blocks every
    // iteration, and cudaFree synchronises the device.  All work on a block is
    // ordered on `stream` (comm work is joined back into it), so reuse needs no
    // further synchronisation.
    std::multimap<size_t, void*> block_cache;
    size_t block_cache_bytes = 0, block_cache_limit = size_t(8) << 30;
    void* take_block_mem(size_t bytes);
    void give_block_mem(void* p, size_t bytes);
    void trim_block_cache();
    void* host_pinned = nullptr;  // small pinned staging
    size_t host_pinned_bytes = 0;
    std::map<GraphKey, GraphEntry> graphs;
    std::map<std::tuple<const void*, int64_t, int>, FilterWorkspace> filter_ws;
    ~Context();
    void* pinned(size_t bytes);
};

// ---- launchers (kernels.cu) ------------------------------------------------------------
enum StepKind {
    kStepSpmmvm = 0,   // Y = (alpha A + beta I) X, beta added iff != 0
    kStepStart2 = 1,   // startup step 2 of apply_filter (filter.hpp:93-103)
    kStepFused = 2,    // spmmvm_fused (kernels.hpp:74-118)
    kStepRecur = 3,    // recurrence_step (kernels.hpp:121-145)
    kStepFusedX2 = 4,  // spmmvm_fused whose X update also carries the previous step's:
                       // X = (X + c_{n-1} V_{n-1}) + c_n V_n (the previous step ran as kStepRecur)
    kStepFusedX3 = 5,  // ... the previous two steps': X = ((X + c_{n-2} V_{n-2}) + c_{n-1} V_{n-1})
                       // + c_n V_n (both ran as kStepRecur)
};

struct StepArgs {
    int kind_step;
    const Matrix* a;
    int64_t width_cols;      // block width in columns
    int64_t row0, row1;      // owned-row range processed by this launch
    const void* in;          // gathered operand, extended-row base
    void* w;                 // W (in/out) or Y (out); owned base
    void* x;                 // X (in/out) owned base, or null
    void* x0;                // x0 for moments (read; written in kStepSpmmvm copy mode)
    double alpha, beta;      // (2alpha, 2beta) already doubled for fused/recur/start2
    double c0, c1, c2;       // start2 combination / fused coeff in c0
    const double* coeff_dev; // fused: device coefficient array (graph-friendly) or null
    int coeff_index;
    int dots_mode;           // 0 none, 1 <x_old, w> (Kahan, complex), 2 Re<x0, w>, 3 m0+m1 (spmmvm start)
    void* dots_out;          // device output (S[nb] for mode 1, double[nb] for 2, 2*nb for 3)
    int partial_base;        // first partial slot of this launch
    bool final_launch;       // this launch reduces all partials [0, partial_base + grid)
    int* grid_used;          // out: number of blocks used
    bool pdl_ok;             // may launch as a programmatic dependent of the previous kernel
};
void launch_step(Context& ctx, const StepArgs& s, cudaStream_t st);
// per-layout step dispatch (step_c.cu / step_r2.cu / step_r1.cu): units = 16- or 8-byte
// units per row
void launch_step_c(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch);
void launch_step_r2(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch);
void launch_step_r1(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch);
// row-group step kernel (step_gc.cu / step_gr2.cu / step_gr1.cu): false = does not apply
// to this launch (nothing launched)
bool launch_group_c(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch);
bool launch_group_r2(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch);
bool launch_group_r1(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch);
// site-ring step kernel (step_ringc.cu): false = does not apply to this launch
bool launch_ring_c(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch);
// group gi of tile t of a grouped matrix -> its first row (linear or line-interleaved tiles)
struct TileMap {
    int64_t line_rows;  // 0: linear
    int lines;          // lattice lines per tile
    int64_t tpl;        // tiles per line group (x blocks)
    CFD_HD int64_t first_row(int64_t t, int gi) const {
        if (line_rows == 0) return t * kTileRows + gi * kGroupRows;
        const int64_t lg = t / tpl, xb = t - lg * tpl;
        const int xs = kTileGroups / lines;  // sites per tile line
        const int xi = gi / lines, yi = gi - xi * lines;
        return lg * lines * line_rows + yi * line_rows + (xb * xs + xi) * kGroupRows;
    }
};
inline TileMap tilemap_of(const GroupedMatrix& g) {
    return TileMap{g.il_line_rows, g.il_lines,
                   g.il_line_rows ? g.il_line_rows / (kGroupRows * (kTileGroups / g.il_lines)) : 1};
}
// grouped form of a device CSR (group.cu); leaves m.grp.ok = false where it does not apply
void build_grouped(Context& ctx, Matrix& m, const int64_t* d_offs, const int64_t* d_cols,
                   const void* d_vals, cudaStream_t st);
// column-slab launches launch_step will use for s (an upper bound: >= the real count)
int step_slab_count(const Context& ctx, const StepArgs& s);
// Steps coeff_index and coeff_index+1 of apply_filter's fused loop in one
// wavefront launch (pair.cu); s.in = U, s.w = W as for the first step.
// Returns false (nothing launched) where the pair kernel does not apply.
bool launch_step_pair(Context& ctx, const StepArgs& s, cudaStream_t st);

// cache a copy of a's values multiplied by s (used by the v3 step kernel)
void ensure_scaled_values(Context& ctx, Matrix& a, double s, cudaStream_t st);
void launch_axpy(Context& ctx, Block& x, const Block& u, const Block& w, double c0, double c1,
                 double c2, cudaStream_t st);
// out[k] = sum_i f(x_ik, y_ik) over owned rows; mode 0: conj(x) y (S), 1: |x|^2 (double)
void launch_column_reduce(Context& ctx, const Block& x, const Block& y, int mode, void* dev_out,
                          cudaStream_t st);
// out[k] = || av_k - lambda_k v_k ||^2 (double)
void launch_residual_sq(Context& ctx, const Block& av, const Block& v, const double* lambda_dev,
                        void* dev_out, cudaStream_t st);
// x(:,k) /= d[k] (d on the device)
void launch_scale_columns(Context& ctx, Block& b, const double* d_dev, cudaStream_t st);
// w <- w - h q (single column, h real or complex)
void launch_axpy_scalar(Context& ctx, Block& w, const Block& q, double hr, double hi,
                        cudaStream_t st);
void launch_copy_columns(Context& ctx, Block& dst, int64_t d0, const Block& src, int64_t s0,
                         int64_t n, cudaStream_t st);
void launch_philox_normal(Context& ctx, Block& b, uint64_t seed, cudaStream_t st);
// dst row i = src row idx[i] (device index list), rows of row_bytes
void launch_gather_rows(Context& ctx, void* dst, const void* src, const int64_t* idx, int64_t n,
                        int64_t row_bytes, cudaStream_t st);
// SELL build from a device CSR (global column indices -> extended-row index)
void build_sell(Context& ctx, Matrix& m, const int64_t* d_offs, const int64_t* d_cols,
                const void* d_vals, cudaStream_t st);

// ---- host helpers (host.cpp) --------------------------------------------------------------
struct HostCsr {
    int kind = 0;
    int64_t dim = 0, row_begin = 0, rows = 0;
    std::vector<int64_t> offs, cols;  // offs relative to row_begin
    std::vector<double> vals;         // interleaved for complex
};
HostCsr gen_graphene(const chebfd_lattice& s, int64_t r0, int64_t r1);
// bitwise Hermitian test of a whole CSR (every (i,j,v) has (j,i,conj v); no duplicate columns)
bool csr_is_hermitian(int kind, int64_t dim, const int64_t* offs, const int64_t* cols,
                      const double* vals);
// moment doubling (DMODE 4) raw sums -> moments: rows q >= 2 become 2 raw - m(q mod 2)
void moments_from_doubling(double* m, int64_t rows, int64_t width);
HostCsr gen_topological_insulator(const chebfd_lattice& s, int64_t r0, int64_t r1);
void validate_lattice(const chebfd_lattice& s, bool needs_z);
// std::mt19937_64 + std::normal_distribution stream (block_vector.hpp:42-51):
// entries [first, first+count) of the row-major global block
void host_randomize(int kind, uint64_t seed, int64_t first, int64_t count, void* out);
// The same stream generated piecewise: emit() ranges in increasing order reuse
// the chunk bookkeeping of earlier calls (jump-ahead + parallel polar method).
class NormalStream {
  public:
    explicit NormalStream(uint64_t seed);
    ~NormalStream();
    void emit(int kind, int64_t first, int64_t count, void* out);
    // entries per emit() call that keep every host thread busy
    static int64_t parallel_piece(int kind);

  private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};
std::vector<double> window_coeffs(double tlo, double thi, double blo, double bhi, int degree);
std::vector<double> kernel_coeffs(int kind, int mu, int degree);
double dos_count(const double* mu, int order, double blo, double bhi, double lo, double hi);
double dos_density(const double* mu, int order, double blo, double bhi, double lambda);
struct HostCsr;
// Halos of rows [r0, r1) derived from the global columns they read (ring
// distance decides lower vs upper neighbour); starts[q] = first row of rank q.
Partition plan_rows(const HostCsr& csr, int64_t r0, int64_t r1, const std::vector<int64_t>& starts);
// The same partition with compact halo lists (see Partition::compact).
Partition plan_rows_compact(const HostCsr& csr, int64_t r0, int64_t r1,
                            const std::vector<int64_t>& starts);
// Extended-row index of global column g under a partition (compact lists searched),
// -2 if the rank holds no copy.
int64_t map_column(const Partition& p, int64_t g);
// Send ranges from every rank's (halo_lo, halo_hi, lo_rank, hi_rank) (all4).
void plan_sends(Partition& p, int rank, int nranks, const int64_t* all4);
// filter design (design.cpp, restating filter_design.cpp)
struct DesignOut {
    int np_opt = 0, predicted_iters = 0;
    double eta_opt = 0, sigma = 0, predicted_mvms = 0, delta_prime = 0, n_target_estimate = 0;
    bool below_recommended = false;
};
double quality_of(int degree, double sigma);
double damping_factor(double tlo, double thi, double dprime, double blo, double bhi, int degree,
                      int kind, int mu);
DesignOut optimize_degree(double tlo, double thi, double dprime, double blo, double bhi, int kind,
                          int mu, double epsilon);
double invert_search_margin(const double* mu, int order, double blo, double bhi, double tlo,
                            double thi, double n_search);
DesignOut choose_parameters(const double* mu, int order, double blo, double bhi, double tlo,
                            double thi, double n_search, int kind, int kmu, double epsilon);
// plane partition of `dim` rows into nranks parts, boundaries on multiples of `plane`
void plane_partition(int64_t dim, int64_t plane, int rank, int nranks, int64_t* r0, int64_t* r1);
// first row of every rank for the lattice models (TI z-planes, graphene y-rows)
void lattice_starts(const chebfd_lattice& s, bool ti, int nranks, std::vector<int64_t>& starts);

}  // namespace cfd
