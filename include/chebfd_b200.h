/* chebfd_b200 -- B200-native ChebFD hot path behind a plain C ABI.
 *
 * This is the drop-in boundary.  The reference has no FFI; its
 * boundary is the C++ template API in /root/reference/proj/include/chebfd/ headers
 * instantiated for double and std::complex<double>.  Each entry point below
 * names the reference function it replaces (file:line relative to
 * /root/reference/proj).  include/chebfd_b200.hpp restores the reference's
 * C++ signatures and exception types on top of this header.
 *
 * Conventions
 *  - Every function returns int status: CHEBFD_OK (0) or a code naming the
 *    reference exception type; chebfd_last_error() returns the message
 *    (thread-local).
 *  - kind: CHEBFD_REAL64 = double, CHEBFD_COMPLEX128 = std::complex<double>
 *    (interleaved re,im), scalar.hpp:12.
 *  - Block vectors are D x nb ROW-MAJOR (entry (i,k) at i*nb+k), exactly the
 *    reference contract block_vector.hpp:15-16, on the device.
 *  - Host buffers are plain pointers; nothing in this header uses torch types.
 *  - A context drives one GPU on one stream.  Not thread-safe per context.
 *    A distributed context (chebfd_ctx_create_dist) row-partitions matrices
 *    and blocks across ranks (one process per GPU) and exchanges halos and
 *    reductions with NCCL.
 */
#ifndef CHEBFD_B200_H
#define CHEBFD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: map to the reference's exception types ---------------- */
enum {
    CHEBFD_OK = 0,
    CHEBFD_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument: shape, alias, degree */
    CHEBFD_ERR_RUNTIME = 2,          /* std::runtime_error: numerical failure */
    CHEBFD_ERR_DOMAIN = 3,           /* std::domain_error */
    CHEBFD_ERR_OUT_OF_RANGE = 4,     /* std::out_of_range */
    CHEBFD_ERR_CUDA = 5,             /* CUDA runtime / cuBLAS / cuSOLVER failure */
    CHEBFD_ERR_NCCL = 6,             /* NCCL failure */
    CHEBFD_ERR_UNSUPPORTED = 7
};

enum { CHEBFD_REAL64 = 0, CHEBFD_COMPLEX128 = 1 };                     /* scalar.hpp:12 */
enum { CHEBFD_PERIODIC_XY_OPEN_Z = 0, CHEBFD_PERIODIC_ALL = 1, CHEBFD_OPEN_ALL = 2 }; /* models.hpp:13 */
enum { CHEBFD_KERNEL_NONE = 0, CHEBFD_KERNEL_FEJER = 1, CHEBFD_KERNEL_JACKSON = 2,
       CHEBFD_KERNEL_LANCZOS = 3 };                                     /* filter.hpp:12 */

typedef struct chebfd_ctx chebfd_ctx;
typedef struct chebfd_matrix chebfd_matrix;
typedef struct chebfd_block chebfd_block;

/* Message of the last failing call on this thread. */
const char* chebfd_last_error(void);
/* Library version string. */
const char* chebfd_version(void);
/* Build features (bit mask): CHEBFD_FEATURE_EXPERIMENTAL = the opt-in kernel variants
 * that measured slower than the default path (CHEBFD_OPT_PAIR != 0, CHEBFD_OPT_KERNEL
 * = 2) are compiled in; without it setting them fails with CHEBFD_ERR_UNSUPPORTED. */
enum { CHEBFD_FEATURE_EXPERIMENTAL = 1 };
int chebfd_build_features(void);

/* ---- context --------------------------------------------------------------- */
/* Single-GPU context on `device` (replaces the OpenMP runtime, parallel.hpp:18-54).
 * One CUDA device per process (one process per GPU): creating a context on a second
 * device while contexts on another exist fails with CHEBFD_ERR_UNSUPPORTED; several
 * contexts on the same device are allowed. */
int chebfd_ctx_create(int device, chebfd_ctx** out);
/* Distributed context: this process is `rank` of `nranks`, one GPU each; the
 * 128-byte NCCL unique id comes from chebfd_nccl_unique_id() on rank 0 and is
 * broadcast by the caller (torch.distributed or MPI). */
int chebfd_nccl_unique_id(unsigned char id[128]);
int chebfd_ctx_create_dist(int device, int rank, int nranks, const unsigned char id[128],
                           chebfd_ctx** out);
int chebfd_ctx_destroy(chebfd_ctx* ctx);
int chebfd_ctx_synchronize(chebfd_ctx* ctx);
/* cudaStream_t the context launches on (for CUDA-event timing by callers). */
int chebfd_ctx_stream(chebfd_ctx* ctx, void** stream);
int chebfd_ctx_info(chebfd_ctx* ctx, int* device, int* rank, int* nranks, int* num_sms);
/* Number of kernels this library launched on ctx since creation (graph
 * replays count every captured kernel). */
int chebfd_ctx_launch_count(chebfd_ctx* ctx, int64_t* count);
/* Options: CHEBFD_OPT_GRAPHS (1 = capture apply_filter into cached CUDA
 * graphs, default 1); CHEBFD_OPT_OVERLAP (1 = overlap the halo exchange with
 * interior rows, default 1); CHEBFD_OPT_KERNEL (step kernel variant: 0 plain
 * register gathers; 1 TMA-staged SELL chunks with pre-scaled values, and the
 * two-units-per-thread kernel for rows of <= 8 entries -- default; 2 also the
 * gathered rows staged in shared memory (experimental); 3 the two-units kernel
 * wherever it applies).  All variants give bit-identical rows. */
/* CHEBFD_OPT_SLAB_UNITS (step kernels sweep the block in column slabs of at
 * most this many 16-byte units; 0 = 256, the measured best -- narrower slabs
 * re-read the matrix per slab).  Changing any option drops captured filters. */
/* CHEBFD_OPT_PAIR (default 0): apply_filter runs two fused steps per launch as a
 * wavefront over the rows that keeps the intermediate vector in L2 (0 off;
 * 1 where the whole filter state is L2-resident; 2 wherever it applies:
 * single-rank operators, rows of <= 16 entries, rows of <= 256 16-byte units).
 * Bit-identical to two single steps.  CHEBFD_OPT_PAIR_TILE_ROWS / _THREADS /
 * _EXTRA tune its tile rows, CTA threads and extra lag tiles (0/0/-1: auto);
 * CHEBFD_OPT_PAIR_HINTS (default 1) sets its L2 eviction-priority hints;
 * CHEBFD_OPT_PAIR_SLAB its column-slab width in 16-byte units (0: the widest
 * slab whose wavefront fits the L2). */
enum { CHEBFD_OPT_GRAPHS = 1, CHEBFD_OPT_OVERLAP = 2, CHEBFD_OPT_KERNEL = 3,
       CHEBFD_OPT_SLAB_UNITS = 5, CHEBFD_OPT_PAIR = 6, CHEBFD_OPT_PAIR_TILE_ROWS = 7,
       CHEBFD_OPT_PAIR_THREADS = 8, CHEBFD_OPT_PAIR_EXTRA = 9, CHEBFD_OPT_PAIR_HINTS = 10,
       CHEBFD_OPT_PAIR_SLAB = 11, CHEBFD_OPT_MOMENTS = 12, CHEBFD_OPT_PDL = 14,
       CHEBFD_OPT_DELAYED_X = 15, CHEBFD_OPT_BAND_BYTES = 16, CHEBFD_OPT_ASYNC_START = 17,
       CHEBFD_OPT_TILES_PER_CTA = 18, CHEBFD_OPT_COMPACT_HALO = 19, CHEBFD_OPT_GRAM = 20,
       CHEBFD_OPT_GROUPED = 21, CHEBFD_OPT_GROUP_LINES = 22, CHEBFD_OPT_RING = 23,
       CHEBFD_OPT_RING_SEGX = 24, CHEBFD_OPT_RING_NO = 25, CHEBFD_OPT_RING_NZ = 26,
       CHEBFD_OPT_RING_ROWS = 27, CHEBFD_OPT_RING_CONSTS = 28,
       CHEBFD_OPT_RING_TMAP = 29, CHEBFD_OPT_RING_ORDER = 30, CHEBFD_OPT_RING_UNIT = 31,
       CHEBFD_OPT_RING_DOTS = 32 };
/* CHEBFD_OPT_RING: the site-ring step kernel (csrc/step_ring.cuh) on complex TI lattice
 * operators with blocks of a multiple of 32 columns: a producer warp stages each x-column of
 * a strip of four lattice lines (site blocks, z -+ 1 rows, matrix values) in shared-memory
 * rings by TMA bulk copies, consumer warps multiply straight from shared memory, so a site
 * block crosses L2 -> SM about once instead of once per referencing site.  Dot-free fused /
 * V_n-only steps; W and X bit-identical to the other step kernels.  1 (default): lattices
 * whose z-plane of the block reaches 2 x CHEBFD_OPT_BAND_BYTES (C4: 1 GB planes), and from a
 * quarter of that (8 MB) on where the grid is a dozen waves of CTAs (TI 64^3); 2: every
 * applicable launch; 0: off (the row-group / SELL kernels).
 * CHEBFD_OPT_RING_SEGX (x-columns per CTA; default 0 = 64, halved down to 16 while the grid
 * would be fewer than 24 waves of CTAs), _NO / _NZ (ring depths, default
 * 5 / 3), _ROWS (rows of a site per consumer thread: 4, 2 or 1; default 2 -- 4 / rows
 * consumer groups share a site's staged operands), _CONSTS (default 1: where every static
 * site of a pattern holds the same off-diagonal values -- the lattice models' hopping terms
 * -- the products take them as kernel-parameter constants and only the four diagonal values
 * per site are read; the builder compares the stored values bit for bit), _TMAP (tensor-map
 * TMA: a site's four rows / a z -+ 1 row pair of a column slab as one 2D box copy; 1 =
 * for slabs narrower than the row (default), 2 = always, 0 = per-row 1D bulk copies), _ORDER
 * (CTA order: 0 bands of strips with x segments fastest, 1 x segments slowest, 2 planes fastest
 * then strips then x segments, 3 = automatic (default): 2 on shallow slabs, else 0; _UNIT: CTAs
 * per band of order 1), _DOTS (default 1: the V_n-only steps that carry the doubling moment
 * sums -- apply_filter with moments, kpm_dos -- also run the site-ring kernel when the step is
 * one launch; per-CTA partials reduced in CTA index order, bitwise reproducible; 0: those
 * steps keep the row-group / SELL kernels). */
/* CHEBFD_OPT_GROUPED (default 1): dot-free steps that run in the band tile order (lattice
 * operators whose z-planes exceed the L2 budget, CHEBFD_OPT_BAND_BYTES) use the row-group
 * kernel: four consecutive rows -- a lattice site's orbitals -- share one merged list of
 * gathered rows, sites of the TI stencil run straight-line code with two multiplies per
 * purely real / imaginary matrix entry.  W and X are bit-identical to the SELL kernels for
 * finite inputs (see csrc/group_patterns.hpp for the sign of exact zeros).  2: every step
 * on every operator with a grouped form (tests); 0: the SELL kernels only.
 * CHEBFD_OPT_GROUP_LINES (default 1; set before building matrices): tiles of the grouped
 * form span 1, 2 or 4 lattice lines (measured: no gain from 2 or 4). */
/* CHEBFD_OPT_GRAM (default 1): gram / SVQB / Rayleigh-Ritz X^H Y of complex blocks of
 * 48+ columns on the library's own FP64 tensor-core (DMMA) kernel -- split-K over the
 * rows, only the upper half of Hermitian products (Y^H Y; Q^H A Q of a Hermitian A);
 * real or narrower blocks on cuBLAS D/ZGEMM.  0 = cuBLAS everywhere, 2 = the DMMA
 * kernel everywhere (even real widths). */
/* CHEBFD_OPT_COMPACT_HALO (default 1; set before building distributed matrices): halos of
 * structurally symmetric operators (the lattice models, bitwise-Hermitian from_csr input)
 * hold only the neighbour rows the local rows reference -- TI reads orbitals {0,3} of the
 * plane below and {1,2} of the plane above, half the plane -- packed on the sender by a
 * gather kernel; 0 = whole contiguous neighbour planes. */
/* CHEBFD_OPT_TILES_PER_CTA (default 2): band-ordered launches run a non-persistent grid
 * of this many consecutive tiles per CTA, dispatched in order by the hardware (a compact
 * wavefront; persistent CTA-strided grids drift apart and lose the band's L2 reuse);
 * 0 = no band order. */
/* CHEBFD_OPT_ASYNC_START (default 2^26): chebfd_solve with n_search given generates the
 * start block (solver.cpp:147-154) on a helper thread, overlapped with the Lanczos
 * bounds and the KPM DOS, when local rows x n_search >= this many entries (0: never).
 * The block is the same stream either way (BlockVector::randomize, bit-identical). */
/* CHEBFD_OPT_BAND_BYTES (default 16 MiB): dot-free step launches on TI lattice operators
 * whose z-plane of the gathered block exceeds 4x this many bytes sweep the rows in bands
 * of lattice lines, plane by plane inside a band (a band slice of the block is at most
 * this size), on a non-persistent grid (CHEBFD_OPT_TILES_PER_CTA), so the z -+ 1
 * neighbour rows are reused from L2; 0 = row order.  Results are identical (row-local
 * arithmetic; launches with dots keep the persistent row-order grid). */
/* CHEBFD_OPT_DELAYED_X (default 3): apply_filter's fused loop updates X once per G
 * steps (G = 2 or 3; 0 / 1: every step) -- the first G-1 steps of a group compute V_n
 * only, the last adds c_{n-2} V_{n-2}, c_{n-1} V_{n-1}, c_n V_n to X, the reference's
 * roundings in its order (kernels.hpp:106) -- so X streams once per G steps; results
 * are bit-identical. */
/* CHEBFD_OPT_PDL: step kernels launch as programmatic dependents of the previous
 * kernel (griddepcontrol), so each step's launch and set-up overlap the previous step's
 * tail -- 1 (default) on small single-rank operators (fewer than 4 x SMs row tiles,
 * where launches dominate), 2 on every single-rank operator, 0 never. */
/* CHEBFD_OPT_MOMENTS: how apply_filter and kpm_dos form <x0, T_n(h) x0>: 0 one
 * dot product against the kept x0 per step (the reference's way, filter.hpp:86-113,
 * spectral.cpp:186-195); 1 (default) where the operator is bitwise Hermitian, the
 * Chebyshev doubling identities T_2n = 2 T_n^2 - 1, T_2n+1 = 2 T_n T_n+1 - T_1: dots of
 * the recurrence vectors already in registers, no x0 stream, and only the first half of
 * the steps reduce (KPM: half the recurrence steps).  Equal up to rounding. */
/* step launches that ran in the band tile order (CHEBFD_OPT_BAND_BYTES) so far */
int chebfd_ctx_band_launches(chebfd_ctx* ctx, int64_t* count);
/* step launches that ran the row-group kernel (CHEBFD_OPT_GROUPED) so far */
int chebfd_ctx_group_launches(chebfd_ctx* ctx, int64_t* count);
/* step launches that ran the site-ring kernel (CHEBFD_OPT_RING) so far */
int chebfd_ctx_ring_launches(chebfd_ctx* ctx, int64_t* count);
int chebfd_ctx_set_option(chebfd_ctx* ctx, int option, int64_t value);

/* CUDA-event timing on the context stream: 16 event slots per context. */
int chebfd_ctx_event_record(chebfd_ctx* ctx, int slot);
/* Milliseconds between two recorded slots (synchronises on slot b). */
int chebfd_ctx_event_elapsed(chebfd_ctx* ctx, int slot_a, int slot_b, float* ms);

/* Pinned host memory for end-to-end transfers. */
int chebfd_host_alloc(size_t bytes, void** out);
int chebfd_host_free(void* p);

/* ---- lattice models (models.hpp:19-29, models.cpp) ------------------------- */
typedef struct {
    int64_t lx, ly, lz; /* lattice size; graphene ignores lz */
    double t;           /* hopping amplitude */
    double disorder;    /* V: box disorder on [-V/2, V/2] (full width) */
    int boundary;       /* CHEBFD_PERIODIC_XY_OPEN_Z etc. */
    uint64_t seed;      /* mt19937_64 seed for the site potentials */
} chebfd_lattice;

/* Host CSR of rows [row_begin, row_end) of the graphene / topological
 * insulator Hamiltonian, bit-identical to graphene() (models.cpp:142-178) /
 * topological_insulator() (models.cpp:80-140) built by the reference's
 * Builder (sparse_matrix.hpp:57-84), but generated stencil-direct (no
 * std::map).  Two-call pattern: with offs == NULL only *nnz (and *dim) are
 * returned; then pass arrays of (row_end-row_begin)+1 / nnz / nnz (values
 * double or interleaved complex).  offs are relative to row_begin. */
int chebfd_csr_graphene(const chebfd_lattice* spec, int64_t row_begin, int64_t row_end,
                        int64_t* dim, int64_t* nnz, int64_t* offs, int64_t* cols, void* vals);
int chebfd_csr_topological_insulator(const chebfd_lattice* spec, int64_t row_begin,
                                     int64_t row_end, int64_t* dim, int64_t* nnz, int64_t* offs,
                                     int64_t* cols, void* vals);

/* ---- distributed row partition (host-only planning) --------------------------- */
/* One process per GPU: contiguous row ranges on lattice planes (TI z-planes,
 * graphene y-rows); gathered blocks live in an extended row space
 * [halo_lo | owned | halo_hi].  The reference has no distribution; this
 * restates the paper's GHOST row distribution. */
typedef struct {
    int64_t dim, row_begin, local_rows;
    int64_t halo_lo, halo_hi;           /* rows received from lo / hi neighbour */
    int64_t lo_src_begin, hi_src_begin; /* first global row of each halo */
    int lo_rank, hi_rank;               /* -1: none */
    int64_t bnd_lo, bnd_hi;             /* rows [0,bnd_lo) / last bnd_hi read a halo */
    int64_t send_lo_begin, send_lo_n;   /* local rows sent to lo_rank */
    int64_t send_hi_begin, send_hi_n;   /* local rows sent to hi_rank */
} chebfd_partition;
/* Plan rank `rank` of `nranks` for a lattice model (0 graphene, 1 TI): rows
 * and halos; send ranges stay zero until chebfd_plan_sends. */
int chebfd_plan_partition(const chebfd_lattice* spec, int model, int rank, int nranks,
                          chebfd_partition* out);
/* Fill the send ranges from every rank's (halo_lo, halo_hi, lo_rank, hi_rank),
 * all4[4*nranks] (what the device path all-gathers over NCCL). */
int chebfd_plan_sends(chebfd_partition* p, int rank, int nranks, const int64_t* all4);
/* Extended-row index of global column g, or -2 if this rank holds no copy. */
int64_t chebfd_plan_map_column(const chebfd_partition* p, int64_t g);

/* ---- device sparse matrix (SELL-C-sigma, C = 32, sigma = 1) ----------------- */
/* From a full host CSR (SparseMatrix ctor + validate, sparse_matrix.hpp:22-100).
 * In a distributed context every rank passes the full matrix and keeps its
 * row partition. */
int chebfd_matrix_from_csr(chebfd_ctx* ctx, int kind, int64_t dim, const int64_t* row_offsets,
                           const int64_t* col_indices, const void* values, chebfd_matrix** out);
/* Stencil-direct device matrices of the two lattice models.  In a
 * distributed context each rank generates only its rows, partitioned on
 * lattice planes (TI z-planes, graphene y-rows). */
int chebfd_matrix_graphene(chebfd_ctx* ctx, const chebfd_lattice* spec, chebfd_matrix** out);
int chebfd_matrix_topological_insulator(chebfd_ctx* ctx, const chebfd_lattice* spec,
                                        chebfd_matrix** out);
int chebfd_matrix_destroy(chebfd_matrix* a);
typedef struct {
    int kind;
    int64_t dim;          /* global dimension D */
    int64_t nnz;          /* global nonzeros (reference count, padding excluded) */
    int64_t local_rows;   /* rows owned by this rank */
    int64_t row_begin;    /* first global row owned */
    int64_t local_nnz;    /* nonzeros in owned rows */
    int64_t sell_entries; /* stored SELL slots incl. padding */
    int64_t halo_lo, halo_hi; /* halo rows received from the lower / upper neighbour */
    int chunk;            /* SELL chunk height C */
    int max_row_len;
    int stage_rows;       /* largest per-chunk gathered-row union of the staged plan (0: none) */
} chebfd_matrix_info;
int chebfd_matrix_get_info(const chebfd_matrix* a, chebfd_matrix_info* out);

/* ---- block vectors (block_vector.hpp:17-102) -------------------------------- */
/* A block conforming to matrix `a` (owned rows of this rank), width nb, zero-filled. */
int chebfd_block_create(chebfd_matrix* a, int64_t width, chebfd_block** out);
/* A free-standing block of `dim` rows (single-GPU contexts). */
int chebfd_block_create_dim(chebfd_ctx* ctx, int kind, int64_t dim, int64_t width,
                            chebfd_block** out);
/* A zero-filled block with the rows (and partition / halos) of `like` and `width`
 * columns -- what the reference's BlockVector<S>(x.dim(), m) builds inside
 * block_mult_small / svqb_orthonormalize (kernels.hpp:216-232, solver.cpp:52-58). */
int chebfd_block_create_like(const chebfd_block* like, int64_t width, chebfd_block** out);
int chebfd_block_destroy(chebfd_block* b);
int chebfd_block_info(const chebfd_block* b, int* kind, int64_t* rows, int64_t* width,
                      int64_t* row_begin);
int chebfd_block_upload(chebfd_block* b, const void* host_rowmajor);
int chebfd_block_download(const chebfd_block* b, void* host_rowmajor);
int chebfd_block_copy(chebfd_block* dst, const chebfd_block* src);
int chebfd_block_zero(chebfd_block* b);
/* BlockVector::randomize (block_vector.hpp:42-51): the same mt19937_64 +
 * libstdc++ normal_distribution stream over the GLOBAL D x nb block, so a
 * distributed block equals the reference's rows. Host-generated, uploaded. */
int chebfd_block_randomize(chebfd_block* b, uint64_t seed);
/* Host: entries [first, first+count) of that stream for a global block of
 * kind `kind` (row-major; complex entries interleaved), generated in parallel
 * with mt19937_64 jump-ahead, bit-identical to the reference. */
int chebfd_host_randomize(int kind, uint64_t seed, int64_t first, int64_t count, void* out);
/* Device Gaussian fill (Philox counter RNG) -- fast synthetic inputs for
 * benchmarks; NOT the reference's stream. */
int chebfd_block_randomize_device(chebfd_block* b, uint64_t seed);
/* x(:,k) *= s[k] for k < width (used to normalise columns). */
int chebfd_block_scale_columns(chebfd_block* b, const double* s);
/* dst(:, d0:d0+n) = src(:, s0:s0+n) */
int chebfd_block_copy_columns(chebfd_block* dst, int64_t d0, const chebfd_block* src, int64_t s0,
                              int64_t n);
int chebfd_block_device_ptr(chebfd_block* b, void** ptr);

/* ---- on-disk formats (matrix_market.cpp, block_vector.hpp:63-96) -------------- */
/* Matrix Market coordinate reader (read_matrix_market, matrix_market.cpp:98-115):
 * real / integer / complex fields, general / symmetric / hermitian storage
 * (mirrored entries added, conjugated for hermitian), duplicates summed in file
 * order, 1-based indices.  Host CSR out (ascending columns).  Call with
 * offs == NULL to get kind / dim / nnz, then again with arrays of dim+1, nnz
 * and nnz (x2 for complex) entries.  *hermitian = storage != general.
 * Errors: CHEBFD_ERR_RUNTIME (banner, field, symmetry, size line, short file),
 * CHEBFD_ERR_OUT_OF_RANGE (index outside [1, D]). */
int chebfd_read_matrix_market(const char* path, int* kind, int64_t* dim, int64_t* nnz,
                              int64_t* offs, int64_t* cols, void* vals, int* hermitian);
/* write_matrix_market (matrix_market.cpp:63-95): lower triangle when hermitian
 * != 0, 17 significant digits (exact round trip). */
int chebfd_write_matrix_market(const char* path, int kind, int64_t dim, const int64_t* offs,
                               const int64_t* cols, const void* vals, int hermitian);
/* Read a Matrix Market file straight into a device SELL matrix (== read + from_csr). */
int chebfd_matrix_from_matrix_market(chebfd_ctx* ctx, const char* path, chebfd_matrix** out);
/* .cbfd block dumps (BlockVector::save/load): u32 magic 0x44464243 "CBFD",
 * u64 D, u32 nb, u32 kind (0 real, 1 complex), D*nb row-major scalars.
 * Raw host-buffer form; data == NULL on load reads only the header.
 * Errors: CHEBFD_ERR_RUNTIME ("bad header", "scalar kind mismatch",
 * "truncated payload", cannot open). */
int chebfd_cbfd_save(const char* path, int kind, uint64_t dim, uint32_t width, const void* data);
int chebfd_cbfd_load(const char* path, int* kind, uint64_t* dim, uint32_t* width, void* data);
/* Device-block forms (single-GPU contexts; a distributed block gives
 * CHEBFD_ERR_UNSUPPORTED).  load creates a block conforming to `a`. */
int chebfd_block_save(const chebfd_block* b, const char* path);
int chebfd_block_load(chebfd_matrix* a, const char* path, chebfd_block** out);

/* ---- kernels (kernels.hpp) ---------------------------------------------------- */
/* Y = (alpha A + beta I) X                                  kernels.hpp:45-69 */
int chebfd_spmmvm(chebfd_matrix* a, chebfd_block* x, chebfd_block* y, double alpha, double beta);
/* W <- 2(alpha A + beta I) U - W;  X <- X + coeff W;  optional dots_k =
 * <x_k(before), w_k(after)> into host `dots` (S[nb]) or NULL.  kernels.hpp:71-118 */
int chebfd_spmmvm_fused(chebfd_matrix* a, chebfd_block* u, chebfd_block* w, chebfd_block* x,
                        double alpha, double beta, double coeff, void* dots);
/* W <- 2(alpha A + beta I) U - W                              kernels.hpp:120-145 */
int chebfd_recurrence_step(chebfd_matrix* a, chebfd_block* u, chebfd_block* w, double alpha,
                           double beta);
/* X <- c0 X + c1 U + c2 W                                     kernels.hpp:147-162 */
int chebfd_block_axpy_scal(chebfd_block* x, const chebfd_block* u, const chebfd_block* w,
                           double c0, double c1, double c2);
/* d_k = <x_k, y_k> -> host S[nb]                               kernels.hpp:194-213 */
int chebfd_column_dots(const chebfd_block* x, const chebfd_block* y, void* out);
/* ||x_k|| -> host double[nb]                                    kernels.hpp:234-240 */
int chebfd_column_norms(const chebfd_block* x, double* out);
/* G(k,l) = <x_k, y_l> -> host row-major S[nx*ny]               kernels.hpp:164-192 */
int chebfd_gram(const chebfd_block* x, const chebfd_block* y, void* out);
/* Y = X B, B host row-major S[nb x bcols], Y width bcols         kernels.hpp:215-232 */
int chebfd_block_mult_small(const chebfd_block* x, const void* b, int64_t bcols, chebfd_block* y);

/* ---- filter (filter.hpp, filter.cpp) ----------------------------------------- */
int chebfd_window_coeffs(double target_lo, double target_hi, double bounds_lo, double bounds_hi,
                         int degree, double* out);                    /* filter.cpp:43-56 */
int chebfd_kernel_coeffs(int kernel, int mu, int degree, double* out); /* filter.cpp:58-84 */
/* combined[0..degree] = g_n c_n, alpha = 2/(b-a), beta = (a+b)/(a-b)   filter.cpp:86-99 */
int chebfd_make_filter(double target_lo, double target_hi, double bounds_lo, double bounds_hi,
                       int degree, int kernel, int mu, double* combined, double* alpha,
                       double* beta);
int chebfd_eval_scalar(const double* combined, int degree, double alpha, double beta,
                       double bounds_lo, double bounds_hi, double x, double* out); /* :101-114 */
/* X <- p[A] X in exactly degree*nb column spMVMs (filter.hpp:73-116).  If
 * moments != NULL it receives m(n,k) = Re<x0_k, T_n(h) x0_k>, (degree+1) x nb
 * row-major (MomentTable, filter.hpp:61-68). */
int chebfd_apply_filter(chebfd_matrix* a, chebfd_block* x, const double* combined, int degree,
                        double alpha, double beta, double* moments);
/* Same, end to end from a HOST block (row-major, owned rows): H2D, filter, D2H. */
int chebfd_apply_filter_host(chebfd_matrix* a, void* x_host, int64_t width,
                             const double* combined, int degree, double alpha, double beta,
                             double* moments);

/* Streamed end-to-end filtering of a sequence of HOST blocks (no reference
 * counterpart: the reference filters in place in host memory).  Job k's
 * H2D copy runs on its own stream while job k-1 filters and job k-2's result
 * copies back, so a stream of filter applications runs at the device rate,
 * not at device + PCIe time.  Two device slots of nb columns; submit() returns
 * once the work is queued: host_in must stay valid until its H2D copy ran and
 * host_out until wait() (pinned memory from chebfd_host_alloc for full-speed
 * copies; host_in == host_out is allowed).  Results are bit-identical to
 * chebfd_apply_filter_host. */
typedef struct chebfd_filter_pipe chebfd_filter_pipe;
int chebfd_filter_pipe_create(chebfd_matrix* a, int64_t width, chebfd_filter_pipe** out);
int chebfd_filter_pipe_submit(chebfd_filter_pipe* p, const void* host_in, void* host_out,
                              const double* combined, int degree, double alpha, double beta);
/* submit + the Rayleigh-Ritz Gram G = X^H X of the filtered block (gram(X, X),
 * kernels.hpp:165-192; row-major width x width scalars, summed over ranks) copied to
 * gram_host with the block; both valid after chebfd_filter_pipe_wait. */
int chebfd_filter_pipe_submit_gram(chebfd_filter_pipe* p, const void* host_in, void* host_out,
                                   const double* combined, int degree, double alpha,
                                   double beta, void* gram_host);
int chebfd_filter_pipe_wait(chebfd_filter_pipe* p);
int chebfd_filter_pipe_destroy(chebfd_filter_pipe* p);

/* ---- solver (solver.hpp / solver.cpp) ------------------------------------------- */
/* SVQB (solver.cpp:32-61): q receives the rank orthonormal columns first. */
int chebfd_svqb(chebfd_block* y, double drop_tol, chebfd_block* q, int64_t* rank);
/* Rayleigh-Ritz (solver.cpp:63-91): v = Ritz vectors; values ascending. */
int chebfd_rayleigh_ritz(chebfd_matrix* a, chebfd_block* q, chebfd_block* v, double* values,
                         double* residual_norms);

/* ---- spectral probes (spectral.cpp) --------------------------------------------- */
int chebfd_lanczos_bounds(chebfd_matrix* a, int iters, uint64_t seed, double* lo,
                          double* hi);                                 /* :96-154 */
/* mu[0..order] raw KPM moments (spectral.cpp:156-205) */
int chebfd_kpm_dos(chebfd_matrix* a, double bounds_lo, double bounds_hi, int order,
                   int num_samples, uint64_t seed, double* mu);
/* Jackson-damped count integral (ChebSeriesDensity::count, spectral.cpp:46-57) */
int chebfd_dos_count(const double* mu, int order, double bounds_lo, double bounds_hi, double lo,
                     double hi, double* out);
/* Jackson-damped density at lambda (ChebSeriesDensity::density, spectral.cpp:31-44) */
int chebfd_dos_density(const double* mu, int order, double bounds_lo, double bounds_hi,
                       double lambda, double* out);
/* weight_density (spectral.cpp:81-88): mu[n] = sum_k moments[n * width + k], n = 0..degree.
 * Errors (invalid_argument): empty moment table. */
int chebfd_weight_density(const double* moments, int degree, int64_t width, double* mu);

/* ---- bench front end (bench.hpp / bench.cpp) ------------------------------------- */
/* BenchPoint (bench.hpp:49-58): model flops and traffic (bench.cpp:28-34, S_i = 4)
 * over the measured seconds per filter application. */
typedef struct {
    int n_b;
    double seconds;    /* per apply_filter (device events, incl. the y = x copy as timed there) */
    double flops;      /* per_row_flops * D * n_b * degree */
    double gflops;
    double gbs_proxy;  /* model traffic / seconds */
    double intensity;  /* I(n_b) */
    double roofline;   /* P* = I(n_b) * b, Gflop/s */
    double efficiency; /* gflops / roofline */
} chebfd_bench_point;
/* intensity_model (bench.cpp:37-41): I(n_b) flop/byte of one blocked step.
 * Errors (invalid_argument): n_b < 1, n_nzr <= 0. */
int chebfd_intensity_model(double n_nzr, int s_d, int s_i, int f_a, int f_m, int n_b,
                           double* out);
/* bandwidth_probe_min_bytes (bench.cpp:42): 8 x the last-level cache (the GPU's L2). */
int chebfd_bandwidth_probe_min_bytes(chebfd_ctx* ctx, uint64_t* out);
/* bandwidth_probe (bench.cpp:44-67) on HBM: read-only streaming reduction over
 * size_bytes (>= the minimum, else CHEBFD_ERR_INVALID_ARGUMENT), max(reps, 5)
 * sweeps timed with CUDA events, median GB/s. */
int chebfd_bandwidth_probe(chebfd_ctx* ctx, uint64_t size_bytes, int reps, double* gbs);
/* bench_filter (bench.cpp:71-126): window = central 10 % of lanczos_bounds(a, 30),
 * Lanczos-2, start block randomize(7); per block size one untimed application
 * (kernel loading + graph capture), then the reference's protocol: one timed
 * warm-up application, repeated (y = x; apply) until >= 0.1 s.  bandwidth_gbs <= 0 runs the probe;
 * *bandwidth_used receives b.  points[n_sizes].  Errors (invalid_argument):
 * degree < 16, empty sweep, n_b < 1. */
int chebfd_bench_filter(chebfd_matrix* a, const int* block_sizes, int n_sizes, int degree,
                        double bandwidth_gbs, chebfd_bench_point* points, double* bandwidth_used);

/* ---- filter design (filter_design.hpp / filter_design.cpp) ------------------------ */
typedef struct {
    int np_opt;              /* optimal degree N_p */
    double eta_opt;          /* spMVMs per vector per decade of damping */
    double sigma;            /* damping factor of the optimal filter */
    double predicted_mvms;   /* eta_opt * (-log10 eps) */
    int predicted_iters;     /* ceil(log10 eps / log10 sigma) */
    double delta_prime;      /* search margin used */
    double n_target_estimate;
    int below_recommended_search_space; /* N_S < 1.25 N_T */
} chebfd_design;
/* damping_factor (filter_design.cpp:178-184) for the window on [tlo,thi] with
 * search margin delta' inside [blo,bhi] */
int chebfd_damping_factor(double target_lo, double target_hi, double delta_prime,
                          double bounds_lo, double bounds_hi, int degree, int kernel, int mu,
                          double* sigma);
/* optimize_degree (filter_design.cpp:204-277) */
int chebfd_optimize_degree(double target_lo, double target_hi, double delta_prime,
                           double bounds_lo, double bounds_hi, int kernel, int mu, double epsilon,
                           chebfd_design* out);
/* invert_search_margin (filter_design.cpp:330-354) from raw KPM moments */
int chebfd_invert_search_margin(const double* mu, int order, double bounds_lo, double bounds_hi,
                                double target_lo, double target_hi, double n_search,
                                double* delta_prime);
/* choose_parameters (filter_design.cpp:356-369) from raw KPM moments */
int chebfd_choose_parameters(const double* mu, int order, double bounds_lo, double bounds_hi,
                             double target_lo, double target_hi, double n_search, int kernel,
                             int kernel_mu, double epsilon, chebfd_design* out);

/* ---- full ChebFD driver (solver.cpp:93-214) ------------------------------------- */
typedef struct {
    double target_lo, target_hi;
    double epsilon;         /* 1e-10 */
    int n_search;           /* 0 = 2*ceil(N_T estimate) */
    int degree;             /* 0 = choose_parameters (filter_design.cpp:356-369) */
    int kernel, kernel_mu;  /* Lanczos, 2 */
    int max_iters;          /* 40 */
    uint64_t seed;          /* 1 */
    int dos_moments;        /* 2000 */
    int dos_samples;        /* 32 */
    double bounds_lo, bounds_hi; /* lo >= hi: Lanczos bounds */
    int collect_weight_density;  /* 1 */
} chebfd_solver_options;

void chebfd_solver_options_default(chebfd_solver_options* o);

typedef struct {
    int converged, iterations, n_search, degree, n_values;
    double total_spmvms, sigma, eta, bounds_lo, bounds_hi, matrix_norm_est, n_target_estimate;
    double seconds, weight_integral;
    /* wall seconds per phase: Lanczos bounds, KPM DOS, filter design, all
     * apply_filter calls, SVQB (incl. rank repair), Rayleigh-Ritz, start block
     * (randomize + normalise) */
    double t_bounds, t_dos, t_design, t_filter, t_ortho, t_rr, t_start;
} chebfd_solve_report;

/* values/residual_norms/accepted: capacity `cap` >= n_search; history:
 * max_iters x 5 (iteration, min_residual, max_residual, accepted,
 * cumulative_spmvms) or NULL; weight_moments: (degree+1) or NULL (summed
 * moments of the last filter, WeightDensity input); vectors: if non-NULL
 * receives a new block with the final Ritz vectors. */
int chebfd_solve(chebfd_matrix* a, const chebfd_solver_options* opts, chebfd_solve_report* rep,
                 int cap, double* values, double* residual_norms, int* accepted,
                 double* history, chebfd_block** vectors);
/* chebfd_solve plus the report's weight density (ConvergenceReport::weight, solver.cpp:
 * 158-162): weight_moments[0..degree] = weight_density(moments of the last filter).mu
 * (spectral.cpp:81-88), *weight_len = degree + 1 (0 when collect_weight_density = 0);
 * weight_cap < degree + 1 is CHEBFD_ERR_INVALID_ARGUMENT. */
int chebfd_solve_ex(chebfd_matrix* a, const chebfd_solver_options* opts, chebfd_solve_report* rep,
                    int cap, double* values, double* residual_norms, int* accepted,
                    double* history, chebfd_block** vectors, int weight_cap,
                    double* weight_moments, int* weight_len);

/* ---- virtual rank groups (vgroup.cu) --------------------------------------------- */
/* The distributed filter's nranks ranks (z-plane row partition, halos, interior /
 * boundary launches, cross-launch dot reduction) driven in lockstep by one host thread
 * on ONE device: rank r's halo rows are pulled from the neighbours' blocks by a gather
 * kernel on its comm stream, ordered by events (no kernel waits on another), and the
 * whole filter can be captured as one CUDA graph.  Results equal the single-rank
 * path's bit for bit (row-local arithmetic); moments, dots and Gram matrices are summed
 * over ranks in rank order.  Used to exercise and time the multi-rank device path where
 * only one GPU exists.  Rank contexts come from chebfd_vgroup_context; blocks are
 * created per rank from the rank's matrix (chebfd_block_create). */
typedef struct chebfd_vgroup chebfd_vgroup;
int chebfd_vgroup_create(int device, int nranks, chebfd_vgroup** out);
int chebfd_vgroup_destroy(chebfd_vgroup* g);
int chebfd_vgroup_context(chebfd_vgroup* g, int rank, chebfd_ctx** out);
/* CHEBFD_OPT_GRAPHS: one graph for all ranks' steps; other options go to every rank */
int chebfd_vgroup_set_option(chebfd_vgroup* g, int option, int64_t value);
/* out[nranks]: rank r's partition of the lattice model (0 graphene, 1 TI) */
int chebfd_vgroup_matrix_lattice(chebfd_vgroup* g, int model, const chebfd_lattice* spec,
                                 chebfd_matrix** out);
/* apply_filter over all ranks (a[r], x[r]); moments: (degree+1) x nb summed over ranks */
int chebfd_vgroup_apply_filter(chebfd_vgroup* g, chebfd_matrix* const* a, chebfd_block* const* x,
                               const double* combined, int degree, double alpha, double beta,
                               double* moments);
/* spmmvm_fused over all ranks; dots (Kahan per rank) summed over ranks */
int chebfd_vgroup_spmmvm_fused(chebfd_vgroup* g, chebfd_matrix* const* a, chebfd_block* const* u,
                               chebfd_block* const* w, chebfd_block* const* x, double alpha,
                               double beta, double coeff, void* dots);
/* gram(X, Y) summed over ranks */
int chebfd_vgroup_gram(chebfd_vgroup* g, chebfd_block* const* x, chebfd_block* const* y,
                       void* out);
/* halo rows received (lo, hi) and rows sent (lo, hi) by a distributed matrix's rank */
int chebfd_vgroup_halo_rows(chebfd_matrix* a, int64_t* halo_lo, int64_t* halo_hi,
                            int64_t* send_lo, int64_t* send_hi);

#ifdef __cplusplus
}
#endif
#endif /* CHEBFD_B200_H */
