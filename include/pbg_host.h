/*
 * pbg_host.h — host-side input preparation for the PB-SpGEMM benchmarks
 * (C-ABI, OpenMP, no device work). Not on the hot path: it builds the CSC/CSR
 * inputs the reference builds with coo_to_csc/coo_to_csr
 * (proj/src/convert.cpp:41-98) from the reference's generators
 * (proj/src/generate.cpp:20-90), plus the benchmark configs' extras
 * (U[0,1) values, RMAT self-loop removal, the 27-point stencil).
 */
#ifndef PBG_HOST_H
#define PBG_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* SplitMix64::next (generate.hpp:21-26) and split_seed (generate.hpp:38-40) */
uint64_t pbgh_split_seed(uint64_t seed, uint64_t stream);

/* gen_er draws (generate.cpp:20-54): n*d (row, col) pairs, column-major in
 * generation order. */
int pbgh_gen_er(int scale, uint32_t d, uint64_t seed, uint32_t* rows, uint32_t* cols);

/* gen_rmat draws before dedup (generate.cpp:56-81): (ef << scale) pairs. */
int pbgh_gen_rmat(int scale, uint32_t ef, uint64_t seed, double a, double b, double c,
                  uint32_t* rows, uint32_t* cols);

/* COO -> CSR. combine: 0 = sum duplicates (coo_to_csr, convert.cpp:41-70),
 * 1 = collapse duplicates to one entry of value 1.0 (gen_rmat's dedup,
 * generate.cpp:83-88). drop_diag removes (i,i). vals may be NULL (1.0).
 * rowptr[nrows+1], colids/vals_out sized nnz (upper bound); *nnz_out gets
 * the result count. */
int pbgh_coo_to_csr(uint32_t nrows, uint32_t ncols, uint64_t nnz, const uint32_t* rows,
                    const uint32_t* cols, const double* vals, int combine, int drop_diag,
                    uint64_t* rowptr, uint32_t* colids, double* vals_out, uint64_t* nnz_out);

/* CSR -> CSC of the same matrix (column-major storage, rows ascending). */
int pbgh_csr_to_csc(uint32_t nrows, uint32_t ncols, const uint64_t* rowptr,
                    const uint32_t* colids, const double* vals, uint64_t* colptr,
                    uint32_t* rowids, double* vals_out);

/* vals[p] = U[0,1) of entry (row, colids[p]):
 * SplitMix64(split_seed(vseed, row<<32|col)).next_unit(). */
int pbgh_csr_fill_values(uint64_t vseed, uint32_t nrows, const uint64_t* rowptr,
                         const uint32_t* colids, double* vals);

/* 27-point stencil on an nx*ny*nz grid, Dirichlet truncation, diagonal 26,
 * off-diagonal -1, in CSR. Pass rowptr=NULL to get only *nnz_out. */
int pbgh_stencil27(uint32_t nx, uint32_t ny, uint32_t nz, uint64_t* rowptr, uint32_t* colids,
                   double* vals, uint64_t* nnz_out);

/* Row band [r0, r1) of a CSC matrix as its own CSC (rows renumbered from 0):
 * the row-slab one GPU multiplies in the row-band partitioning. Pass
 * colptr_out=NULL to size: *nnz_out gets the slab's nnz. */
int pbgh_csc_row_band(uint32_t nrows, uint32_t ncols, const uint64_t* colptr,
                      const uint32_t* rowids, const double* vals, uint32_t r0, uint32_t r1,
                      uint64_t* colptr_out, uint32_t* rowids_out, double* vals_out,
                      uint64_t* nnz_out);

/* Per-row flop of A*B from CSC A and CSR B (for band cuts), row_flop[nrows]. */
int pbgh_row_flop(uint32_t nrows, uint32_t ncols, const uint64_t* a_colptr,
                  const uint32_t* a_rowids, const uint64_t* b_rowptr, uint64_t* row_flop);

/* Flop-balanced cuts of [0, nrows) into g bands: cuts[0]=0, cuts[g]=nrows. */
int pbgh_band_cuts(uint32_t nrows, const uint64_t* row_flop, uint32_t g, uint32_t* cuts);

/* ---- Matrix Market I/O (mm_read / mm_write, proj/src/mmio.cpp:33-130) ----
 * Coordinate format; real/integer/pattern fields, general/symmetric
 * symmetry. Symmetric storage is expanded to both triangles (diagonal kept
 * single, the mirror entry right after its source); pattern entries get 1.0;
 * 1-based indices leave 0-based; entries keep file order. Malformed input
 * fails with the reference's parse_error message ("name:line: what"),
 * available from pbgh_last_error(). Two calls: open parses the file into a
 * handle and reports dims and entry count, fetch copies the entries out. */
typedef struct pbgh_mm pbgh_mm;
int pbgh_mm_open(const char* path, pbgh_mm** out, uint32_t* nrows, uint32_t* ncols,
                 uint64_t* nnz);
int pbgh_mm_fetch(const pbgh_mm* h, uint32_t* rows, uint32_t* cols, double* vals);
void pbgh_mm_free(pbgh_mm* h);
/* coordinate real general, values printed round-trip exact (%.17g). */
int pbgh_mm_write(const char* path, uint32_t nrows, uint32_t ncols, uint64_t nnz,
                  const uint32_t* rows, const uint32_t* cols, const double* vals);
/* Message of the last non-zero return on this thread. */
const char* pbgh_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* PBG_HOST_H */
