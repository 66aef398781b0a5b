/*
 * pbg.h — C-ABI of the B200-native PB-SpGEMM hot path.
 *
 * C = A * B with A in CSC and B in CSR, C in CSR: outer-product expand into
 * row-range bins, per-bin sort + duplicate merge, CSR assembly — the path of
 * spgemm::pb_multiply (reference: proj/include/spgemm/pb_spgemm.hpp:116,
 * proj/src/pb_spgemm.cpp:330-361), re-implemented as sm_100a CUDA kernels.
 *
 * The reference has no FFI layer: its boundary is the C++ call
 *     spgemm::PbResult spgemm::pb_multiply(const CscMatrix&, const CsrMatrix&,
 *                                          const PbConfig& = {});
 * This header is what that C++ entry point is re-implemented on top of
 * (include/spgemm_b200/pb_spgemm.hpp, the drop-in); INTEGRATION.md shows the
 * binding. Plain pointers and sizes only: no torch, no CUDA types.
 *
 * No CPU fallback: without a CUDA device every compute entry point returns
 * PBG_ERR_NODEVICE.
 */
#ifndef PBG_H
#define PBG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes. The C++ drop-in maps DIM/NBINS/LBIN/FLOP_OVERFLOW to
 * spgemm::parameter_error (reference types.hpp:80-83, pb_spgemm.cpp:88-89,
 * :103-105, :252-253), INTERNAL to spgemm::internal_error (types.hpp:89-91,
 * pb_spgemm.cpp:241-245, :342-345, :358-359) and the rest to
 * std::runtime_error. */
enum {
    PBG_OK = 0,
    PBG_ERR_DIM = 1,            /* a.ncols != b.nrows              (types.hpp:97-102)  */
    PBG_ERR_NBINS = 2,          /* cfg.nbins not a power of two    (pb_spgemm.cpp:88)  */
    PBG_ERR_LBIN = 3,           /* lbin_bytes not k*16, k>0        (pb_spgemm.cpp:252) */
    PBG_ERR_FLOP_OVERFLOW = 4,  /* flop does not fit 64 bits       (pb_spgemm.cpp:103) */
    PBG_ERR_INTERNAL = 5,       /* a conservation self-check failed                    */
    PBG_ERR_CUDA = 6,
    PBG_ERR_OOM = 7,
    PBG_ERR_NCCL = 8,
    PBG_ERR_ARG = 9,            /* null pointer / malformed view                        */
    PBG_ERR_UNIMPLEMENTED = 10,
    PBG_ERR_NODEVICE = 11
};

/* A borrowed compressed-sparse view. For CSC: nrows x ncols, ptr = colptr
 * [ncols+1], idx = rowids [nnz]; for CSR: ptr = rowptr [nrows+1], idx = colids.
 * Field meaning follows spgemm::CscMatrix / CsrMatrix (types.hpp:51-69):
 * u64 offsets, u32 indices, f64 values. */
typedef struct pbg_csx_view {
    uint32_t nrows;
    uint32_t ncols;
    uint64_t nnz;
    const uint64_t* ptr;
    const uint32_t* idx;
    const double* val;
} pbg_csx_view;

/* spgemm::PbConfig (pb_spgemm.hpp:11-17) plus GPU fields. The reference
 * fields keep their validation contract; on the GPU nbins/l2_bytes/
 * balanced_bins only shape the REFERENCE-layout symbolic report
 * (pbg_symbolic_fetch), nthreads and lbin_bytes' staging role have no GPU
 * meaning. The GPU bins are sized to shared memory. */
typedef struct pbg_config {
    uint32_t nbins;        /* 0 = auto (choose_nbins), else a power of two */
    uint32_t lbin_bytes;   /* must be a positive multiple of 16            */
    uint64_t l2_bytes;     /* reference L2 sizing input (default 1 MiB)     */
    int32_t nthreads;      /* ignored on the GPU                           */
    int32_t balanced_bins; /* reference-layout report only                 */
    int32_t device;        /* CUDA ordinal, -1 = current device            */
    uint32_t bin_cap;      /* GPU bin capacity in tuples, 0 = default 4096 */
    /* host path: devices to split C's rows over. 0/1 = the
     * one device `device`; G > 1 = devices device, device+1, ... each taking
     * a flop-balanced row band of A (cut on the device, balanced_starts
     * rule) against all of B; -1 = every visible device. */
    int32_t ngpus;
    uint32_t flags;        /* PBG_FLAG_* */
    /* reserved[0]: cap on tuples per round (0 = from free HBM); above it a
     * device multiplies its rows as flop-balanced bands one after another.
     * reserved[1]: force the number of expand row bands (0 = auto). */
    uint64_t reserved[4];
} pbg_config;

/* pbg_config.flags */
enum {
    /* test hook: with ngpus > the visible device count, bands wrap around the
     * devices (several contexts on one device; bands never wait on each
     * other) so the multi-device path runs on a one-GPU box */
    PBG_FLAG_WRAP_DEVICES = 1
};

/* spgemm::PhaseReport times (report.hpp:26-33) measured with CUDA events,
 * plus the acceptance counters (acceptance.cpp:46-58). t_sort covers the
 * per-bin distinct count, the offset scan and the fused sort+merge+CSR
 * kernel; t_compress and t_convert are 0 (fused). */
typedef struct pbg_report {
    double t_symbolic, t_expand, t_sort, t_compress, t_convert, t_total; /* seconds */
    double t_h2d, t_d2h;  /* host path only                                       */
    uint64_t flop, nnz_c, nnz_a, nnz_b;
    uint64_t tuples_into_sort; /* sum of expand fill cursors                      */
    uint64_t merged_total;     /* sum of per-bin merged counts                    */
    uint32_t nbins;            /* reference-layout bin count (choose_nbins rule) */
    uint32_t gpu_bins;         /* shared-memory bins actually used on the GPU     */
    uint32_t heavy_bins;       /* bins larger than bin_cap (global-memory path)   */
    uint32_t bin_cap;
    uint64_t tuple_bytes;      /* bytes of tuple storage (12 B per tuple + pad)   */
    uint64_t sort_fallbacks;   /* bins sorted by the LSD fallback (clustered keys) */
    uint32_t expand_bands;     /* row bands the expand ran in (L2 write frontier) */
    uint32_t pad0;
    double t_count;            /* per-bin distinct-key count + offset scan (in t_sort) */
    double t_sortmerge_kernel; /* the sort+merge+CSR kernel alone (in t_sort)     */
    uint32_t ngpus;            /* devices the row bands ran on (host path)        */
    uint32_t nrounds;          /* most bounded-memory rounds on one device        */
    double t_device_max;       /* slowest device: its bands' t_total summed       */
    double t_device_min;       /* fastest device                                  */
} pbg_report;

typedef struct pbg_handle pbg_handle;
typedef struct pbg_context pbg_context;

/* Thread-local message for the last non-zero return on this thread. */
const char* pbg_last_error(void);
void pbg_default_config(pbg_config* cfg);
/* 1 when a CUDA device is usable, else 0. */
int pbg_device_available(void);

/* ---- host-buffer path: the drop-in for pb_multiply ------------------- */
/* Copies A (CSC) and B (CSR) from host memory, runs the pipeline and keeps C
 * on the device. *nnz_c receives nnz(C) so the caller can size its arrays. */
int pbg_multiply_begin(const pbg_csx_view* a_csc, const pbg_csx_view* b_csr,
                       const pbg_config* cfg, pbg_handle** out, uint64_t* nnz_c);
/* D2H of C into caller-owned rowptr[m+1], colids[nnz], values[nnz]; rep may
 * be NULL. */
int pbg_multiply_fetch(pbg_handle* h, uint64_t* rowptr, uint32_t* colids, double* values,
                       pbg_report* rep);
/* One call, C written straight into caller-owned host arrays: rowptr
 * [nrows+1], colids/values of capacity cap entries (pinned memory makes the
 * copies asynchronous). C = A*B is computed as flop-balanced row bands sized
 * to free HBM, each band's copy to the host overlapping the next band's
 * multiply — products whose tuples or C exceed HBM (C3) run without host
 * staging. With cfg.ngpus > 1 the bands run on several devices. Returns
 * PBG_ERR_ARG with *nnz_c = the bands' nnz so far when cap is too small.
 * rep->t_d2h = wall time of the whole call. */
int pbg_multiply_into(const pbg_csx_view* a_csc, const pbg_csx_view* b_csr, const pbg_config* cfg,
                      uint64_t* rowptr, uint32_t* colids, double* values, uint64_t cap,
                      uint64_t* nnz_c, pbg_report* rep);
/* coo_to_csr / coo_to_csc (convert.cpp:41-98) on the GPU, through the same
 * pipeline: the conversion is the product A.B with A(major(e), e) = 1 and
 * B(e, minor(e)) = val(e), so duplicates are summed (exact zeros kept) and
 * minor indices ordered by the sort+merge path. to_csc = 0 gives the CSR
 * (major = row), 1 the CSC (major = col). Entries outside nrows x ncols
 * return PBG_ERR_ARG (validate, convert.cpp:8-37). Host arrays; the result
 * is read with pbg_multiply_fetch (rowptr = the major pointer array) and
 * freed with pbg_release. */
int pbg_coo_convert_begin(uint32_t nrows, uint32_t ncols, uint64_t nnz, const uint32_t* rows,
                          const uint32_t* cols, const double* vals, int to_csc,
                          const pbg_config* cfg, pbg_handle** out, uint64_t* nnz_out);
/* The benchmark inputs of SURVEY.md §8d built on the GPU: gen_er (kind 0,
 * d = ef distinct rows per column) or gen_rmat (kind 1, Graph500 a,b,c,
 * duplicates collapsed, self-loops dropped) with the reference's seeded
 * streams (generate.cpp:20-90), converted like pbg_coo_convert_begin, values
 * U[0,1) from SplitMix64(split_seed(vseed, row << 32 | col)). to_csc = 0
 * gives the CSR, 1 the CSC; read with pbg_multiply_fetch, free with
 * pbg_release. */
int pbg_generate_begin(int kind, int scale, uint32_t ef, uint64_t seed, uint64_t vseed, int to_csc,
                       const pbg_config* cfg, pbg_handle** out, uint64_t* nnz_out);
/* spgemm::hash_multiply (baseline.hpp:21-24, baseline.cpp:141-200) on the
 * GPU: C = A.B with A, B and C in CSC (column Gustavson SpGEMM, one shared-
 * memory hash table per output column, sized bit_ceil(2 f_j) like the
 * reference's). Same errors as pbg_multiply_begin (PBG_ERR_DIM,
 * PBG_ERR_FLOP_OVERFLOW); columns of more than 4096 products (RMAT hubs)
 * use a dense global-memory accumulator (k_hash_hub). Read with
 * pbg_multiply_fetch (rowptr = colptr[b.ncols+1], colids = row ids), free
 * with pbg_release. pbg_report: flop, nnz_c, t_symbolic (column flop +
 * scan), t_sort (hash + sort + compaction), t_total. */
int pbg_hash_multiply_begin(const pbg_csx_view* a_csc, const pbg_csx_view* b_csc,
                            const pbg_config* cfg, pbg_handle** out, uint64_t* nnz_c);
/* The reference SymbolicResult (pb_spgemm.hpp:48-55) on the REFERENCE bin
 * layout: per_column_flop[a.ncols], per_bin_flop[nbins], bin_row_starts
 * [nbins+1]; nbins from pbg_report.nbins. Any pointer may be NULL. */
int pbg_symbolic_fetch(pbg_handle* h, uint64_t* per_column_flop, uint64_t* per_bin_flop,
                       uint32_t* bin_row_starts);
void pbg_release(pbg_handle* h);

/* ---- device-resident path: inputs already in HBM --------------------- */
int pbg_context_create(int device, pbg_context** out);
void pbg_context_destroy(pbg_context* ctx);
/* Views hold DEVICE pointers. stream is a cudaStream_t (NULL = legacy default).
 * Blocks until nnz(C) is known. C stays in the context until the next call. */
int pbg_multiply_device(pbg_context* ctx, const pbg_csx_view* a_csc, const pbg_csx_view* b_csr,
                        const pbg_config* cfg, void* stream, uint64_t* nnz_c, pbg_report* rep);
/* Device pointers to the last product's CSR arrays (valid until the next
 * pbg_multiply_device on this context). */
int pbg_context_result(pbg_context* ctx, const uint64_t** rowptr, const uint32_t** colids,
                       const double** values);
/* Reference-layout symbolic arrays of the last product (host destinations). */
int pbg_context_symbolic(pbg_context* ctx, const pbg_config* cfg, uint64_t* per_column_flop,
                         uint64_t* per_bin_flop, uint32_t* bin_row_starts);
/* Kernel launches issued by the last pbg_multiply_device call. */
uint32_t pbg_context_launches(pbg_context* ctx);

/* ---- row bands on the device (pbg_bands.cuh) ----------- */
/* Flop-balanced cuts of rows [r0, r1) of C = A*B into nbands bands
 * (device-resident A in CSC, B in CSR): cuts[0] = r0, cuts[nbands] = r1,
 * cut j after the first row whose inclusive flop prefix (from r0) reaches
 * j/nbands of the range's flop — the reference's balanced_starts rule
 * (pb_spgemm.cpp:58-82). *flop (may be NULL) = flop of rows [r0, r1).
 * Host destination for cuts. */
int pbg_band_cuts_device(pbg_context* ctx, const pbg_csx_view* a_csc, const pbg_csx_view* b_csr,
                         uint32_t r0, uint32_t r1, uint32_t nbands, void* stream, uint32_t* cuts,
                         uint64_t* flop);
/* The CSC row slab A(r0:r1, :) (rows renumbered from 0) built on the device
 * into caller device arrays colptr[ncols+1], rowids/values[cap]; with
 * colptr == NULL only *nnz is returned (size query). §8f f1: a device's row
 * slab of A without a host pass. */
int pbg_row_slab_device(pbg_context* ctx, const pbg_csx_view* a_csc, uint32_t r0, uint32_t r1,
                        void* stream, uint64_t* colptr, uint32_t* rowids, double* values,
                        uint64_t cap, uint64_t* nnz);
/* C(r0:r1, :) = A(r0:r1, :) * B for device-resident A (the whole CSC) and B:
 * the row slab of A is extracted on the device, the product has r1 - r0 rows
 * (band-local rowptr) and is read with pbg_context_result like a
 * pbg_multiply_device product. */
int pbg_multiply_device_band(pbg_context* ctx, const pbg_csx_view* a_csc, const pbg_csx_view* b_csr,
                             uint32_t r0, uint32_t r1, const pbg_config* cfg, void* stream,
                             uint64_t* nnz_c, pbg_report* rep);
/* Checksum of the context's last product (its own rows numbered from
 * row_base): out[0] = nnz, out[1] = row-count hash, out[2] = (row, col)
 * hash (order-free, sums of mixed words: bands add up to the whole); *vsum =
 * sum of the values. The checksum-and-discard mode of products whose C is
 * kept nowhere (C5b). */
int pbg_context_checksum(pbg_context* ctx, uint64_t row_base, void* stream, uint64_t* out,
                         double* vsum);

/* Development aid (no reference counterpart): the work bins of the context's
 * last product -- the sort kernel's units of work (GPU bins and the key-range
 * pieces of heavy rows): tuples, key bits, flags (bit0 scratch buffer, bit1
 * merged, bit2 heavy sub-bin) and distinct keys of the first min(cap, *nw)
 * work bins; any output array may be NULL. */
int pbg_context_workbins(pbg_context* ctx, uint64_t cap, uint64_t* nw, uint64_t* n,
                         uint32_t* keybits, uint32_t* flags, uint64_t* nnz);

/* ---- reference helpers with no device work --------------------------- */
/* choose_nbins (pb_spgemm.cpp:10-18) */
uint32_t pbg_choose_nbins(uint64_t flop, uint32_t nrows, uint64_t l2_bytes, uint32_t tuple_bytes);

#ifdef __cplusplus
}
#endif
#endif /* PBG_H */
