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
  RDMM_ERR_INVALID = 7         /* std::invalid_argument / bad parameters */
} rdmm_status;

/* Message of the last failure on the calling thread ("" if none). */
const char* rdmm_last_error(void);
/* Library version string and the compiled device architecture. */
const char* rdmm_version(void);

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
 *   RDMM_SPMM_NO_PREFETCH disable the L2 prefetch of the next window's B rows.
 */
#define RDMM_SPMM_C_ZERO 1u
#define RDMM_SPMM_NO_PREFETCH 2u
int rdmm_spmm_csr_ex(int dtype_bytes, uint32_t rows, uint32_t cols, uint32_t n,
                     uint64_t nnz, const uint32_t* row_ptr,
                     const uint32_t* col_idx, const void* val, const void* B,
                     uint64_t ldb, void* C, uint64_t ldc, unsigned flags,
                     void* workspace, size_t workspace_bytes,
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
void rdmm_spgemm_plan_destroy(rdmm_spgemm_plan* plan);
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

#ifdef __cplusplus
}
#endif
#endif /* RDMM_CUDA_H */
