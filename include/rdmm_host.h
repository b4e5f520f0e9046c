/*
 * rdmm_host.h -- C-ABI of the host driver layer (the C++ API in
 * include/rdmm/ headers, instantiated for float and double), so that non-C++
 * callers (the Python mirror, bench.py, an FFI binding) can drive the
 * reference's distributed entry points:
 *
 *   Fabric / FabricConfig           fabric.hpp:205-412
 *   DistSparse / DistDense          distmat.hpp:92-398
 *   init / init_from_global         distmat.hpp:113-145, 240-263
 *   to_global                       distmat.hpp:183-197, 359-377
 *   run_multiply / RunOptions /     algos.hpp:39-96, 673-752
 *   RunReport
 *
 * Collective calls (init*, run_multiply) drive every rank hosted by the
 * calling process (one thread per local rank) and must be made by every
 * process of a multi-process fabric in the same order.
 */
#ifndef RDMM_HOST_H
#define RDMM_HOST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rdmm_h_fabric rdmm_h_fabric;
typedef struct rdmm_h_matrix rdmm_h_matrix;

int rdmm_h_fabric_create(uint32_t nranks, uint64_t heap_bytes,
                         uint32_t node_group, uint64_t queue_capacity,
                         uint32_t first_local, uint32_t nlocal,
                         const int* devices, const char* session,
                         rdmm_h_fabric** out);
void rdmm_h_fabric_destroy(rdmm_h_fabric* f);
void* rdmm_h_fabric_handle(rdmm_h_fabric* f); /* the rdmm_fabric* */

/* kind: 0 sparse (DistSparse), 1 dense (DistDense); dtype_bytes 4|8 */
int rdmm_h_matrix_create(rdmm_h_fabric* f, int kind, int dtype_bytes,
                         uint64_t m, uint64_t n, uint32_t tm, uint32_t tn,
                         uint32_t pr, uint32_t pc, int matrix_id,
                         rdmm_h_matrix** out);
void rdmm_h_matrix_destroy(rdmm_h_matrix* mat);

/* Collective initialisation.  Sparse: a global CSR (host or device
 * pointers; NULL row_ptr = empty tiles).  Dense: a global row-major array
 * with leading dimension ld (host or device pointer; NULL = zeros). */
int rdmm_h_sparse_init(rdmm_h_matrix* mat, const uint32_t* row_ptr,
                       const uint32_t* col_idx, const void* values,
                       uint64_t nnz, int on_device);
int rdmm_h_dense_init(rdmm_h_matrix* mat, const void* global, uint64_t ld);

/* Collective: zero every tile of a dense matrix in place (fresh C). */
int rdmm_h_dense_zero(rdmm_h_matrix* mat);
/* End-to-end download: each local rank copies ITS tiles of the result into
 * the host array (dense: row-major global layout; sparse: the raw CSR arrays
 * of its tiles, concatenated into buf (capacity cap; pinned memory for
 * full speed), *bytes set to the amount moved). */
int rdmm_h_dense_owned_to_host(rdmm_h_matrix* mat, void* global, uint64_t ld);
int rdmm_h_sparse_owned_to_host(rdmm_h_matrix* mat, void* buf, uint64_t cap,
                                uint64_t* bytes);
/* Asynchronous dense download: the copies are enqueued on `stream` (a
 * caller-owned cudaStream_t on the local rank's device, one local rank per
 * process), ordered after the rank's queued compute; returns at once, so a
 * step's download overlaps the next step's upload and multiply. */
int rdmm_h_dense_owned_to_host_async(rdmm_h_matrix* mat, void* global, uint64_t ld,
                                     void* stream);
/* The compute stream of a local rank (timing events go there). */
void* rdmm_h_fabric_stream(rdmm_h_fabric* f, uint32_t rank);

/* Host gathers (verification; bypass traffic accounting). */
int rdmm_h_dense_to_host(rdmm_h_matrix* mat, void* out);
int rdmm_h_sparse_nnz(rdmm_h_matrix* mat, uint64_t* nnz);
int rdmm_h_sparse_to_host(rdmm_h_matrix* mat, uint32_t* row_ptr,
                          uint32_t* col_idx, void* values);

typedef struct {
  int variant; /* 0 summa_bsp .. 5 ws_locality (algos.hpp:18-25) */
  int ws_base;
  int prefetch;
  int offset;
  uint64_t seed;
  double delay_ns_per_flop;
  double random_delay_ms_max;
  int record_events;
  int record_triples;
  int lookahead;
  int ws_local_inplace;
  int checksum;
  int fuse_k;
  int split_local; /* fused stationary-C: local products first on the first tile */
  int time_stages; /* per-k-step device time of each rank's multiplies (stage_ms) */
  int pipeline;    /* narrow fused stationary-C: row-block fetch/concat/SpMM pipeline */
  int row_blocks;  /* row blocks of that pipeline (0 = default) */
  int deterministic; /* reproducible k-order accumulation of narrow dense C tiles */
} rdmm_h_options;

#define RDMM_H_MAX_RANKS 64
typedef struct {
  double wall_seconds;
  double checksum;
  uint64_t total_flops, total_multiplies, total_steals;
  uint32_t nranks;
  uint64_t multiplies[RDMM_H_MAX_RANKS];
  uint64_t flops[RDMM_H_MAX_RANKS];
  uint64_t output_nnz[RDMM_H_MAX_RANKS];
  uint64_t steals[RDMM_H_MAX_RANKS];
  uint64_t steals_local[RDMM_H_MAX_RANKS];
  uint64_t pushes[RDMM_H_MAX_RANKS];
  uint64_t pops[RDMM_H_MAX_RANKS];
  uint64_t bytes_self[RDMM_H_MAX_RANKS];
  uint64_t bytes_on_node[RDMM_H_MAX_RANKS];
  uint64_t bytes_off_node[RDMM_H_MAX_RANKS];
  double total_seconds[RDMM_H_MAX_RANKS];
  uint64_t ntriples;     /* recorded (i,j,k) triples, all local ranks */
  uint32_t* triples;     /* 4 x uint32 per triple: rank, i, j, k (malloc'd) */
  /* Per-rank flops per k tile step (RankStats::stage_flops, the table of
   * analytics.hpp:66-90): nranks x nstages row-major, malloc'd (free with
   * rdmm_h_free); ranks hosted by other processes are zero rows. */
  uint32_t nstages;
  uint64_t* stage_flops;
  /* Per-rank device milliseconds per k tile step (RankStats::stage_ms; with
   * time_stages), same shape and ownership as stage_flops; NULL otherwise. */
  double* stage_ms;
} rdmm_h_report;

int rdmm_h_run_multiply(rdmm_h_fabric* f, rdmm_h_matrix* A, rdmm_h_matrix* B,
                        rdmm_h_matrix* C, const rdmm_h_options* opts,
                        rdmm_h_report* rep);
void rdmm_h_free(void* p);

/* Matrix Market coordinate I/O (replaces rdmm::read_matrix_market /
 * write_matrix_market, mmio.hpp:50-116): plain or gzip input; symmetric
 * files expanded; duplicates summed.  Host CSR arrays are malloc'd (free with
 * rdmm_h_free); dtype_bytes 4 (float) or 8 (double). */
int rdmm_h_read_matrix_market(const char* path, int dtype_bytes, uint32_t* rows,
                              uint32_t* cols, uint64_t* nnz, uint32_t** row_ptr,
                              uint32_t** col_idx, void** values);
int rdmm_h_write_matrix_market(const char* path, int dtype_bytes, uint32_t rows, uint32_t cols,
                               const uint32_t* row_ptr, const uint32_t* col_idx,
                               const void* values);

#ifdef __cplusplus
}
#endif
#endif /* RDMM_HOST_H */
