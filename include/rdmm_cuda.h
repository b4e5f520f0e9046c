/*
 * rdmm_cuda.h -- the drop-in C-ABI of the B200-native rdmm hot path
 * (librdmm_cuda.so).  Plain pointers and sizes; no torch or C++ types.
 *
 * It replaces, entry for entry, the reference's per-tile kernels and its
 * one-sided fabric (paths relative to /root/reference/proj/include/rdmm/):
 *
 *   kernels  tile.hpp:170-307  spmm_local / spgemm_flops / spgemm_local /
 *                              csr_add / dense_add_into
 *   inputs   gen.hpp:20-181    counter RNG, rmat, uniform_tiles,
 *                              random_dense (device-side generators)
 *   fabric   fabric.hpp:205-575 Fabric / RankCtx: symmetric heaps, put/get,
 *                              get_nb/wait, fetch_add, queues, barrier
 *
 * Conventions
 *  - Every entry point returns an rdmm_status (0 = OK) and leaves a message
 *    for rdmm_last_error() (thread-local) on failure.  The codes mirror the
 *    reference exception taxonomy (tile.hpp:19-23, fabric.hpp:38-60,
 *    algos.hpp:98-101).
 *  - Kernel entry points take DEVICE pointers and a CUDA stream
 *    (rdmm_stream_t == cudaStream_t) and are stream-ordered: they enqueue and
 *    return.  index_t is uint32 (tile.hpp:17); dense tiles are row-major with
 *    explicit leading dimensions (tile.hpp:43-55).
 *  - Thread-safe across devices; not re-entrant on one device from several
 *    host threads that share a workspace (pass explicit workspaces then).
 */
#ifndef RDMM_CUDA_H
#define RDMM_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* rdmm_stream_t; /* cudaStream_t */

typedef enum {
  RDMM_OK = 0,
  RDMM_ERR_DIMENSION = 1,      /* dimension_error        tile.hpp:19-23 */
  RDMM_ERR_FABRIC = 2,         /* fabric_error           fabric.hpp:38-41 */
  RDMM_ERR_HEAP_EXHAUSTED = 3, /* heap_exhausted_error   fabric.hpp:43-53 */
  RDMM_ERR_QUEUE_FULL = 4,     /* queue_full_error       fabric.hpp:55-60 */
  RDMM_ERR_PROTOCOL = 5,       /* protocol_error         algos.hpp:98-101 */
  RDMM_ERR_CUDA = 6,           /* CUDA runtime failure */
  RDMM_ERR_INVALID = 7,        /* std::invalid_argument / bad parameters */
  RDMM_ERR_IO = 8              /* mmio_error             mmio.hpp:19-22 */
} rdmm_status;

/* Message of the last failure on the calling thread ("" if none). */
const char* rdmm_last_error(void);
/* Library version string and the compiled device architecture. */
const char* rdmm_version(void);
/* Number of this library's kernels launched so far (process-wide). */
unsigned long long rdmm_kernel_launches(void);
/* Device timing of the hot kernels: when enabled, CUDA events are recorded
 * on the launching stream around each launch (kind 1 = SpMM launch pair,
 * 2 = SpGEMM numeric, 3 = dense accumulate).  _get sums the durations of
 * one kind (-1: all) recorded since the last rdmm_kernel_timing() call. */
void rdmm_kernel_timing(int enable);
int rdmm_kernel_timing_get(int kind, double* total_ms, unsigned long long* count);

/* ------------------------------------------------------------------ SpMM */
/*
 * C += A * B  (reference spmm_local, tile.hpp:170-188).
 *   A: rows x cols CSR (row_ptr[rows+1], col_idx[nnz], val[nnz]); nnz must
 *      equal row_ptr[rows] (the device-resident tile's directory nnz).
 *   B: cols x n row-major, leading dimension ldb;  C: rows x n, ldc.
 * Rows that do not straddle a work-chunk boundary accumulate in the
 * reference's order (k ascending, fused multiply-add starting from C), so
 * they are bit-identical to the reference for any values; straddling rows add
 * their chunk partials in ascending order (deterministic).
 * workspace: NULL (library-managed per thread/device) or at least
 * rdmm_spmm_workspace_bytes(...) bytes of device memory.
 * flops (optional, host): 2*nnz*n, the reference FlopMeter (tile.hpp:185).
 */
size_t rdmm_spmm_workspace_bytes(uint32_t rows, uint64_t nnz, uint32_t n,
                                 int dtype_bytes);
int rdmm_spmm_csr_f32(uint32_t rows, uint32_t cols, uint32_t n, uint64_t nnz,
                      const uint32_t* row_ptr, const uint32_t* col_idx,
                      const float* val, const float* B, uint64_t ldb, float* C,
                      uint64_t ldc, void* workspace, size_t workspace_bytes,
                      rdmm_stream_t stream, uint64_t* flops);
int rdmm_spmm_csr_f64(uint32_t rows, uint32_t cols, uint32_t n, uint64_t nnz,
                      const uint32_t* row_ptr, const uint32_t* col_idx,
                      const double* val, const double* B, uint64_t ldb,
                      double* C, uint64_t ldc, void* workspace,
                      size_t workspace_bytes, rdmm_stream_t stream,
                      uint64_t* flops);
/* Extended form: dtype_bytes 4|8 and flags.
 *   RDMM_SPMM_C_ZERO      C is all-zero on entry (a fresh tile): rows with
 *                         nonzeros are written, C is never read; results are
 *                         identical to the accumulate form on a zero C.
 */
#define RDMM_SPMM_C_ZERO 1u
/*   RDMM_SPMM_NNZ_ON_DEVICE  nnz is only an upper bound: the kernels read the
 *                         real count from row_ptr[rows] on the device (a CSR
 *                         produced by an earlier kernel on the same stream,
 *                         e.g. a row block of rdmm_csr_concat_cols_rows);
 *                         flops is reported as 0. */
#define RDMM_SPMM_NNZ_ON_DEVICE 2u
/*   RDMM_SPMM_ATOMIC     accumulate into C with red.global.add (rows of at most
 *                         31 vectors, the narrow slot kernels; ignored
 *                         otherwise): C is never read, several products into
 *                         the same C may run concurrently; the summation
 *                         order of a row varies between runs (exact for
 *                         integer data, within the fp tolerance otherwise). */
#define RDMM_SPMM_ATOMIC 4u
int rdmm_spmm_csr_ex(int dtype_bytes, uint32_t rows, uint32_t cols, uint32_t n,
                     uint64_t nnz, const uint32_t* row_ptr,
                     const uint32_t* col_idx, const void* val, const void* B,
                     uint64_t ldb, void* C, uint64_t ldc, unsigned flags,
                     void* workspace, size_t workspace_bytes,
                     rdmm_stream_t stream, uint64_t* flops);

/* Fused K-tile form: C += A * [B_0; B_1; ...] where B is given as nseg
 * (<= 16) row segments of seg_rows rows each (the B(k,j) tiles of one tile
 * column, stacked), all with leading dimension ldb.  A's column g reads row
 * g % seg_rows of segment g / seg_rows.  One pass over A and C for the whole
 * tile column (stationary-C with K tiles, algos.hpp:378-415). */
int rdmm_spmm_csr_seg(int dtype_bytes, uint32_t rows, uint32_t n, uint64_t nnz,
                      const uint32_t* row_ptr, const uint32_t* col_idx,
                      const void* val, const void* const* bseg, uint32_t nseg,
                      uint32_t seg_rows, uint64_t ldb, void* C, uint64_t ldc,
                      unsigned flags, void* workspace, size_t workspace_bytes,
                      rdmm_stream_t stream, uint64_t* flops);

/* ---------------------------------------------------------------- SpGEMM */
/*
 * C = sum_t A_t * B_t  over a list of terms, rows x ncols, sorted rows,
 * cancelled zeros kept (reference spgemm_local, tile.hpp:211-255).  A term
 * whose a_row_ptr is NULL is an identity term contributing B_t as-is, so
 *   spgemm_local(a,b)  = { a*b }                          (tile.hpp:211)
 *   csr_add(a,b)       = { I*a, I*b }                     (tile.hpp:257)
 *   stationary-C tile  = { I*C0, A(i,0)B(0,j), ... }      (algos.hpp:250-263)
 * Two calls: rdmm_spgemm_symbolic bins rows, counts distinct columns, writes
 * c_row_ptr (rows+1, device) and returns the output nnz and the reference
 * FlopMeter flops (2 * multiply-adds, tile.hpp:197-209) on the host (it
 * synchronises the stream); the caller allocates col_idx/values of c_nnz and
 * calls rdmm_spgemm_numeric.  Column indices are bit-exact with the
 * reference; values are summed in hardware order (exact for integer-valued
 * data, within rounding otherwise).  All operand pointers are device
 * pointers and must stay valid until rdmm_spgemm_numeric returns.
 * A plan's working buffers live in the per-(device, stream) scratch pool, so
 * they are reused across calls without cudaMalloc: run symbolic and numeric
 * of one plan on the same stream, and do not interleave a second plan's
 * symbolic on that stream between them.
 */
typedef struct {
  const uint32_t* a_row_ptr; /* NULL: identity term */
  const uint32_t* a_col_idx;
  const void* a_val;
  const uint32_t* b_row_ptr;
  const uint32_t* b_col_idx;
  const void* b_val;
} rdmm_spgemm_term;
typedef struct rdmm_spgemm_plan rdmm_spgemm_plan;
int rdmm_spgemm_symbolic(uint32_t rows, uint32_t ncols, int dtype_bytes,
                         const rdmm_spgemm_term* terms, int nterms,
                         uint32_t* c_row_ptr, rdmm_spgemm_plan** plan,
                         uint64_t* c_nnz, uint64_t* flops,
                         rdmm_stream_t stream);
int rdmm_spgemm_numeric(rdmm_spgemm_plan* plan, uint32_t* c_col_idx,
                        void* c_val, rdmm_stream_t stream);
/* Numeric pass with flags.  RDMM_SPGEMM_DETERMINISTIC: values are the
 * reference's for ANY inputs, bitwise and run to run -- each output is the
 * fma chain of its products in the reference's loop order (tile.hpp:225-237),
 * the terms combined in order like successive csr_adds (tile.hpp:257-288);
 * products are expanded and stably sorted per row batch (slower; opt-in). */
#define RDMM_SPGEMM_DETERMINISTIC 1u
int rdmm_spgemm_numeric_ex(rdmm_spgemm_plan* plan, uint32_t* c_col_idx, void* c_val,
                           unsigned flags, rdmm_stream_t stream);
void rdmm_spgemm_plan_destroy(rdmm_spgemm_plan* plan);
/* FlopMeter flops of each term (identity terms count 0). */
int rdmm_spgemm_plan_term_flops(const rdmm_spgemm_plan* plan, uint64_t* out);
/* rows per symbolic / numeric tier (6 each: 5 hash tiers + dense) */
int rdmm_spgemm_plan_info(const rdmm_spgemm_plan* plan, uint32_t* sym_tiers,
                          uint32_t* num_tiers);

/* --------------------------------------------------------- dense accumulate */
/* c[i] += x[i] for i < count (reference dense_add_into, tile.hpp:300-307).
 * 2-D strided form: rows x cols with leading dimensions. */
int rdmm_dense_add_into_f32(uint32_t rows, uint32_t cols, float* c,
                            uint64_t ldc, const float* x, uint64_t ldx,
                            rdmm_stream_t stream);
int rdmm_dense_add_into_f64(uint32_t rows, uint32_t cols, double* c,
                            uint64_t ldc, const double* x, uint64_t ldx,
                            rdmm_stream_t stream);

/* -------------------------------------------------- distributed helpers */
/* Tile (r0.., c0..) of a device-resident global CSR (distmat.hpp:265-282):
 * count writes out_rp (nrows+1) and returns the tile nnz (synchronises);
 * fill copies the column-rebased indices and values. */
int rdmm_csr_extract_count(const uint32_t* row_ptr, const uint32_t* col_idx,
                           uint64_t r0, uint32_t nrows, uint64_t c0,
                           uint32_t ncols, uint32_t* out_rp, uint64_t* nnz,
                           rdmm_stream_t stream);
int rdmm_csr_extract_fill(int dtype_bytes, const uint32_t* row_ptr,
                          const uint32_t* col_idx, const void* val,
                          uint64_t r0, uint32_t nrows, uint64_t c0,
                          uint32_t ncols, const uint32_t* out_rp,
                          uint32_t* out_ci, void* out_val,
                          rdmm_stream_t stream);
/* Concatenate K (<= 16) CSR tiles of the same rows side by side: tile k's
 * columns are offset by k*col_stride (the A(i,0..K-1) tiles of one tile row
 * -> one CSR for the fused K-tile SpMM).  tile_nnz is accepted for
 * compatibility and unused (the output row pointer is computed on the
 * device without a scan or a host round trip).  out_rp has rows+1 entries,
 * out_ci / out_val the sum of the tiles' nnz. */
int rdmm_csr_concat_cols(int dtype_bytes, uint32_t rows, uint32_t K,
                         const uint32_t* const* row_ptr,
                         const uint32_t* const* col_idx,
                         const void* const* values, const uint64_t* tile_nnz,
                         uint64_t col_stride, uint32_t* out_rp, uint32_t* out_ci,
                         void* out_val, rdmm_stream_t stream);
/* The same for the block of rows [r0, r0+rows) of the tiles: a standalone
 * CSR (out_rp[0] = 0) of those rows, e.g. one row block of a pipelined
 * fused stationary-C step.  col_offsets (host, K entries; NULL = k *
 * col_stride) sets the column offset of each tile, e.g. its natural column
 * position when the tiles are concatenated in a rotated order. */
int rdmm_csr_concat_cols_rows(int dtype_bytes, uint32_t r0, uint32_t rows, uint32_t K,
                              const uint32_t* const* row_ptr, const uint32_t* const* col_idx,
                              const void* const* values, uint64_t col_stride,
                              const uint64_t* col_offsets, uint32_t* out_rp, uint32_t* out_ci,
                              void* out_val, rdmm_stream_t stream);
/* Sum of a dense tile's values in double (checksum, algos.hpp:634-669). */
int rdmm_tile_sum(int dtype_bytes, uint32_t rows, uint32_t cols, uint64_t ld,
                  const void* p, rdmm_stream_t stream, double* out);
/* A single-thread kernel spinning ~ns nanoseconds (straggler injection). */
int rdmm_spin_delay(uint64_t ns, rdmm_stream_t stream);

/* ------------------------------------------------------- input generators */
/* Device-side, bit-identical to the reference host generators (gen.hpp). */

/* gen.hpp:20-34 counter RNG, for tests. out[i] = rng::at(seed, first + i). */
int rdmm_gen_rng_at(uint64_t seed, uint64_t first, uint64_t count,
                    uint64_t* out, rdmm_stream_t stream);
/* gen.hpp:174-181: out[i] = T(int(rng::at(seed, i) % (max_value+1))). */
int rdmm_gen_random_dense(uint64_t count, uint64_t seed, int max_value,
                          int dtype_bytes, void* out, rdmm_stream_t stream);
/* Real-valued parity twin: out[i] = 2*u01(seed, i) - 1. */
int rdmm_gen_real_twin(uint64_t count, uint64_t seed, int dtype_bytes,
                       void* out, rdmm_stream_t stream);

/* R-MAT (gen.hpp:58-92) built directly as a device CSR.  Two calls:
 * rdmm_gen_rmat_begin generates + sorts + deduplicates into an internal
 * device buffer and reports nnz; rdmm_gen_rmat_finish writes row_ptr
 * (2^scale + 1), col_idx (nnz) and values (nnz; 1 or multiplicity) into
 * caller buffers and releases the internal state.  Synchronous. */
typedef struct rdmm_gen_state rdmm_gen_state;
int rdmm_gen_rmat_begin(double a, double b, double c, double d,
                        uint32_t scale, uint32_t edgefactor, uint64_t seed,
                        int multiplicity, rdmm_gen_state** st, uint64_t* nnz);
/* uniform_tiles (gen.hpp:97-133), same two-call protocol. */
int rdmm_gen_uniform_tiles_begin(uint64_t m, uint64_t k, uint32_t p, double d,
                                 uint64_t seed, rdmm_gen_state** st,
                                 uint64_t* nnz);
int rdmm_gen_finish(rdmm_gen_state* st, int dtype_bytes, uint32_t* row_ptr,
                    uint32_t* col_idx, void* values);
void rdmm_gen_abort(rdmm_gen_state* st);

/* permute_symmetric (gen.hpp:134-155): P A P^T with the reference's
 * Fisher-Yates permutation over rng::at(seed, i).  Device CSR in, device CSR
 * out (out_row_ptr rows+1, out_col_idx / out_values nnz; caller-owned).
 * RDMM_ERR_DIMENSION if rows != cols.  Synchronous on `stream`. */
int rdmm_permute_symmetric(uint32_t rows, uint32_t cols, uint64_t nnz,
                           const uint32_t* row_ptr, const uint32_t* col_idx,
                           const void* values, int dtype_bytes, uint64_t seed,
                           uint32_t* out_row_ptr, uint32_t* out_col_idx,
                           void* out_values, rdmm_stream_t stream);
/* The permutation alone, on the host: perm[old index] = new index. */
int rdmm_permutation(uint32_t n, uint64_t seed, uint32_t* perm);

/* ================================================================ fabric */
/*
 * The one-sided fabric (reference fabric.hpp:26-575) on B200:
 *  - one DEVICE heap per rank (cudaMalloc on the rank's GPU, first-fit,
 *    8-byte aligned -- fabric.hpp:277-360); every rank's heap is mapped into
 *    every other rank's device address space (peer access inside a process,
 *    CUDA IPC across processes), so a GlobalPtr resolves to a device address
 *    any rank can copy from or load from over NVLink;
 *  - a node-shared CONTROL segment (POSIX shared memory, pinned and mapped
 *    into every rank's device): fetch-add cells, remote queues, the barrier
 *    and the abort flag live here, so a reservation is one host atomic and a
 *    queue push one host atomic + store;
 *  - ranks are threads of one process (run_ranks, fabric.hpp:556-575) or one
 *    process per GPU (torchrun) sharing the control segment by name.
 * Host threads call these with the rank they act for (`caller`); calls for
 * one rank must come from one thread at a time (fabric.hpp:414-415).
 */
typedef struct rdmm_fabric rdmm_fabric;

/* GlobalPtr (fabric.hpp:30-36).  offset bit 63 set = control-segment cell. */
typedef struct {
  uint32_t rank;
  uint32_t pad_;
  uint64_t offset;
  uint64_t length;
} rdmm_gptr;
#define RDMM_CTRL_BIT (1ull << 63)

typedef struct {
  uint32_t nranks;         /* P (FabricConfig::nranks, fabric.hpp:206) */
  uint32_t node_group;     /* ranks per node group for byte classification */
  uint64_t heap_bytes;     /* device heap per rank (fabric.hpp:207) */
  uint64_t queue_capacity; /* default queue capacity (fabric.hpp:209) */
  uint64_t ctrl_bytes;     /* control arena (0 = default 64 MiB) */
  uint32_t first_local;    /* ranks [first_local, first_local+nlocal) */
  uint32_t nlocal;         /*   are hosted by this process            */
  const int* devices;      /* CUDA device of each local rank (nlocal) */
  const char* session;     /* shm name shared by all processes; NULL or ""
                              when every rank is local */
} rdmm_fabric_config;

int rdmm_fabric_create(const rdmm_fabric_config* cfg, rdmm_fabric** out);
void rdmm_fabric_destroy(rdmm_fabric* f);
uint32_t rdmm_fabric_nranks(const rdmm_fabric* f);
uint32_t rdmm_fabric_node_group(const rdmm_fabric* f);
uint64_t rdmm_fabric_queue_capacity(const rdmm_fabric* f);
int rdmm_fabric_is_local(const rdmm_fabric* f, uint32_t rank);
int rdmm_fabric_device(const rdmm_fabric* f, uint32_t rank); /* local only */
/* Per-local-rank streams owned by the fabric: 0 = compute, 1..2 = copy,
 * 3 = side compute (work overlapped with stream 0, e.g. a pipelined concat). */
rdmm_stream_t rdmm_fabric_stream(rdmm_fabric* f, uint32_t rank, int which);
/* Process-local sequence number (1, 2, ...): processes that create objects
 * in the same order get the same numbers (collective tags). */
uint64_t rdmm_fabric_next_uid(rdmm_fabric* f);
/* Mark a rank failed: wakes every barrier with RDMM_ERR_FABRIC. */
void rdmm_fabric_abort(rdmm_fabric* f, const char* why);

/* Heap (fabric.hpp:235-254, 277-360); rank must be local. */
int rdmm_heap_alloc(rdmm_fabric* f, uint32_t rank, uint64_t nbytes,
                    rdmm_gptr* out);
int rdmm_heap_free(rdmm_fabric* f, rdmm_gptr p);
int rdmm_heap_remaining(const rdmm_fabric* f, uint32_t rank, uint64_t* out);
/* Device address of p as seen from `caller`'s GPU (local or peer-mapped);
 * validates p against the heap (fabric.hpp:316-328). */
int rdmm_gptr_device(rdmm_fabric* f, uint32_t caller, rdmm_gptr p,
                     void** dev);

/* One-sided transfers (fabric.hpp:436-471).  Device-side: stream-ordered
 * copies on `stream` (NULL = the caller's copy stream 1); the handle is a
 * CUDA event that rdmm_wait either makes `consumer` wait on (no host block)
 * or, with consumer NULL, synchronises on the host.  Every transfer is
 * recorded in the traffic log under the caller's phase label. */
typedef struct {
  void* event;
  int error;
} rdmm_handle;
int rdmm_get_nb(rdmm_fabric* f, uint32_t caller, rdmm_gptr src, void* dst,
                rdmm_stream_t stream, rdmm_handle* h);
int rdmm_put_nb(rdmm_fabric* f, uint32_t caller, const void* src,
                rdmm_gptr dst, rdmm_stream_t stream, rdmm_handle* h);
int rdmm_wait(rdmm_fabric* f, rdmm_handle* h, rdmm_stream_t consumer);
/* Blocking host-buffer forms (init / to_global / small headers). */
int rdmm_get_host(rdmm_fabric* f, uint32_t caller, rdmm_gptr src, void* dst);
/* Host read that bypasses the traffic log (Fabric::raw, fabric.hpp:251). */
int rdmm_peek(rdmm_fabric* f, uint32_t caller, rdmm_gptr src, void* dst);
int rdmm_put_host(rdmm_fabric* f, uint32_t caller, const void* src,
                  rdmm_gptr dst);

/* Remote atomic fetch-add on an 8-byte cell (fabric.hpp:473-487). */
int rdmm_fetch_add_i64(rdmm_fabric* f, uint32_t caller, rdmm_gptr cell,
                       int64_t delta, int64_t* old);
/* Control-segment cells: `count` zeroed int64 cells owned by `owner`
 * (WorkGrid storage, algos.hpp:103-133).  Collective over all ranks: every
 * rank passes the same tag and receives the same base pointer. */
int rdmm_ctrl_cells(rdmm_fabric* f, uint32_t caller, uint64_t tag,
                    uint64_t count, rdmm_gptr* base);

/* Remote queues (fabric.hpp:362-375, 502-528): MPMC push, owner-only pop,
 * exactly-once delivery; each entry carries a GlobalPtr plus up to 40 bytes
 * of inline header.  rdmm_queue_open is collective: every rank calls it with
 * the same tag and gets the ids of all P queues (queue r owned by rank r). */
int rdmm_queue_open(rdmm_fabric* f, uint32_t caller, uint64_t tag,
                    uint64_t capacity, uint64_t* qids /* P entries */);
int rdmm_queue_push(rdmm_fabric* f, uint32_t caller, uint64_t qid,
                    rdmm_gptr v, const void* inl, uint32_t inl_bytes);
/* *got = 0 when empty. */
int rdmm_queue_pop(rdmm_fabric* f, uint32_t caller, uint64_t qid,
                   rdmm_gptr* v, void* inl, uint32_t inl_bytes, int* got);
/* Release control-segment storage of the collective with `tag` (queues and
 * cells); collective. */
int rdmm_ctrl_release(rdmm_fabric* f, uint32_t caller, uint64_t tag);

/* Collective barrier over all ranks (fabric.hpp:532): first synchronises
 * the caller's fabric streams, so device work issued before the barrier is
 * complete and visible after it. */
int rdmm_barrier(rdmm_fabric* f, uint32_t caller);

/* Traffic log (fabric.hpp:89-203) -- phase labels, tile fetch records,
 * per-rank event streams (Event, fabric.hpp:62-70). */
void rdmm_set_phase(rdmm_fabric* f, uint32_t caller, int64_t label);
int64_t rdmm_phase(rdmm_fabric* f, uint32_t caller);
void rdmm_record_tile_fetch(rdmm_fabric* f, uint32_t caller, uint32_t owner,
                            int matrix, uint32_t i, uint32_t j);
void rdmm_emit_compute(rdmm_fabric* f, uint32_t caller, uint64_t flops);
/* Record a transfer the caller satisfied without a copy engine: a self
 * alias, or a payload read in place over NVLink by a kernel. */
void rdmm_record_self_get(rdmm_fabric* f, uint32_t caller, uint64_t bytes);
void rdmm_record_get(rdmm_fabric* f, uint32_t caller, uint32_t owner,
                     uint64_t bytes);
typedef struct {
  uint64_t bytes_put, bytes_got, puts, gets, atomic_ops;
} rdmm_traffic;
int rdmm_traffic_pair(const rdmm_fabric* f, uint32_t src, uint32_t dst,
                      rdmm_traffic* out);
int rdmm_traffic_total(const rdmm_fabric* f, rdmm_traffic* out);
void rdmm_traffic_clear(rdmm_fabric* f);
typedef struct {
  uint32_t src, dst;
  int64_t label;
  int32_t matrix;
  uint32_t i, j;
} rdmm_tile_fetch;
/* Copies up to cap records; returns the total count. */
uint64_t rdmm_tile_fetches(const rdmm_fabric* f, rdmm_tile_fetch* out,
                           uint64_t cap);
typedef struct {
  int32_t kind; /* 0 transfer, 1 compute, 2 queue_op */
  uint32_t src, dst;
  uint64_t bytes, flops;
} rdmm_event;
void rdmm_event_sink(rdmm_fabric* f, uint32_t caller, int enable);
uint64_t rdmm_events(const rdmm_fabric* f, uint32_t rank, rdmm_event* out,
                     uint64_t cap);

/* Device memory helpers for the host layer (stream-ordered pool memory on
 * the rank's GPU) so the C++ API needs no CUDA runtime of its own. */
int rdmm_dev_alloc(rdmm_fabric* f, uint32_t rank, uint64_t bytes,
                   rdmm_stream_t stream, void** out);
int rdmm_dev_free(rdmm_fabric* f, uint32_t rank, void* p,
                  rdmm_stream_t stream);
int rdmm_memcpy(void* dst, const void* src, uint64_t bytes,
                rdmm_stream_t stream); /* any direction; NULL stream = sync */
int rdmm_memset(void* dst, int value, uint64_t bytes, rdmm_stream_t stream);
int rdmm_event_record(rdmm_stream_t stream, void** event);
/* Timing-enabled event (per-stage device time, RunOptions::time_stages) and
 * the elapsed milliseconds between two of them (blocks until b completed). */
int rdmm_timing_event_record(rdmm_stream_t stream, void** event);
int rdmm_event_elapsed_ms(void* a, void* b, float* ms);
int rdmm_event_query(void* event, int* done); /* done=1 when complete */
int rdmm_event_wait(void* event, rdmm_stream_t consumer);
int rdmm_event_sync(void* event);
void rdmm_event_destroy(void* event);
int rdmm_stream_sync(rdmm_stream_t stream);
int rdmm_set_device(int device);
int rdmm_get_device(int* device);
int rdmm_device_count(int* n);
/* Strided 2-D copy (any direction), e.g. a dense tile out of a global array. */
int rdmm_memcpy2d(void* dst, uint64_t dpitch, const void* src, uint64_t spitch,
                  uint64_t width_bytes, uint64_t rows, rdmm_stream_t stream);
/* Host address of a control-segment pointer (RDMM_CTRL_BIT set). */
void* rdmm_ctrl_host(rdmm_fabric* f, rdmm_gptr p);

#ifdef __cplusplus
}
#endif
#endif /* RDMM_CUDA_H */
