/*
 * rdmm_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference rdmm CPU algorithms on the SpMM/SpGEMM
 * hot path (reference: /root/reference/proj/include/rdmm/{tile,gen,algos}.hpp).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load this library, and only as the checker or the timed CPU
 * baseline -- never as the product path.
 *
 * Parity is PINNED: tests/test_oracle.py checks every function below against
 * golden vectors produced by the reference itself (oracle/_ref, built from
 * the reference headers by oracle/Makefile; fixtures in tests/golden/ made by
 * tests/golden/make_golden.py) and against the reference's own KATs.
 *
 * dtype codes: 4 = float32, 8 = float64.
 */
#ifndef RDMM_ORACLE_H
#define RDMM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* CSR with uint32 indices (reference index_t, tile.hpp:17). Owned buffers are
 * malloc'd by the oracle and released with orc_csr_free. */
typedef struct {
  uint32_t rows, cols;
  uint64_t nnz;
  int dtype;
  uint32_t* row_ptr; /* rows+1 */
  uint32_t* col_idx; /* nnz */
  void* values;      /* nnz of dtype */
} orc_csr;

/* gen.hpp:20-34 */
uint64_t orc_splitmix64(uint64_t x);
uint64_t orc_rng_at(uint64_t seed, uint64_t counter);
double orc_rng_u01(uint64_t seed, uint64_t counter);

/* gen.hpp:58-92. multiplicity=0 collapses duplicates to 1. Returns 0 / <0. */
int orc_rmat(double a, double b, double c, double d, uint32_t scale,
             uint32_t edgefactor, uint64_t seed, int multiplicity, int dtype,
             orc_csr* out);
/* gen.hpp:97-133 */
int orc_uniform_tiles(uint64_t m, uint64_t k, uint32_t p, double d,
                      uint64_t seed, int dtype, orc_csr* out);
/* gen.hpp:138-155 */
int orc_permute_symmetric(const orc_csr* m, uint64_t seed, orc_csr* out);
/* gen.hpp:158-172 */
int orc_random_csr(uint32_t rows, uint32_t cols, double density, uint64_t seed,
                   int max_value, int dtype, orc_csr* out);
/* gen.hpp:174-181; out holds rows*cols values of dtype, row-major */
void orc_random_dense(uint32_t rows, uint32_t cols, uint64_t seed,
                      int max_value, int dtype, void* out);

/* tile.hpp:70-95: sort (r,c), sum duplicates in sorted order. */
int orc_from_coo(uint32_t rows, uint32_t cols, uint64_t n, const uint32_t* r,
                 const uint32_t* c, const void* v, int dtype, orc_csr* out);

/* tile.hpp:170-188: c += a*b, dense row-major with leading dims. Returns
 * flops (2*nnz*n) or 0 on mismatch (err set to -1). */
uint64_t orc_spmm_local(const orc_csr* a, uint32_t b_rows, uint32_t n,
                        const void* b, uint64_t ldb, void* c, uint64_t ldc,
                        int* err);
/* Row-range restriction of orc_spmm_local (rows [r0,r1)), for bounded CPU
 * baseline samples; same arithmetic. */
uint64_t orc_spmm_rows(const orc_csr* a, uint32_t r0, uint32_t r1, uint32_t n,
                       const void* b, uint64_t ldb, void* c, uint64_t ldc);
/* tile.hpp:197-209 */
uint64_t orc_spgemm_flops(const orc_csr* a, const orc_csr* b);
/* tile.hpp:211-255 (Gustavson, cancelled zeros kept). Rows [r0,r1) of a;
 * r1 = a->rows for the whole product. flops = 2*madds. */
int orc_spgemm_local(const orc_csr* a, const orc_csr* b, uint32_t r0,
                     uint32_t r1, orc_csr* out, uint64_t* flops);
/* tile.hpp:257-288 */
int orc_csr_add(const orc_csr* a, const orc_csr* b, orc_csr* out);
/* tile.hpp:300-307 */
void orc_dense_add_into(uint64_t n, void* c, const void* contrib, int dtype);
/* tile.hpp:105-117 */
int orc_csr_well_formed(const orc_csr* a);

/* algos.hpp:634-650 (dense) and 652-669 (sparse): order-insensitive
 * checksum sum(hash(i,j) * tile_sum). */
double orc_checksum_dense(uint64_t m, uint64_t n, uint32_t tm, uint32_t tn,
                          const void* g, int dtype);
double orc_checksum_sparse(const orc_csr* g, uint32_t tm, uint32_t tn);

void orc_csr_free(orc_csr* a);
void orc_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
