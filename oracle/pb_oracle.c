/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the PB-SpGEMM hot path.
 *
 * A plain-C, single-threaded restatement of the reference's algorithm
 * (arXiv 2002.11302 artifact, /root/reference/proj). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it, and only as the checker or the timed CPU baseline — never as
 * the product path. Parity of this restatement is PINNED against the compiled
 * reference (oracle/_ref, see build_ref.sh) and against the golden fixtures in
 * tests/golden/ made from it (tests/golden/make_golden.py).
 *
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint32_t idx_t;
typedef uint64_t off_t64;

/* ---------------- SplitMix64 (include/spgemm/generate.hpp:12-40) -------- */
static uint64_t sm_next(uint64_t* s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static uint64_t sm_below(uint64_t* s, uint64_t bound) {
    const uint64_t limit = bound * (UINT64_MAX / bound);
    uint64_t x;
    do { x = sm_next(s); } while (x >= limit);
    return x % bound;
}
static double sm_unit(uint64_t* s) { return (double)(sm_next(s) >> 11) * 0x1.0p-53; }
uint64_t orc_split_seed(uint64_t seed, uint64_t stream) {
    uint64_t s = seed ^ (stream * 0xD6E8FEB86659FD93ULL);
    return sm_next(&s);
}

/* U[0,1) value of entry (r, c): SURVEY.md §8d value assignment, built on
 * SplitMix64::next_unit and split_seed (generate.hpp:35-40). */
double orc_value(uint64_t vseed, uint32_t r, uint32_t c) {
    uint64_t s = orc_split_seed(vseed, ((uint64_t)r << 32) | c);
    return sm_unit(&s);
}

/* gen_er (src/generate.cpp:20-54): Floyd sampling of d distinct rows per
 * column. Writes n*d (row, col) pairs in generation order. */
void orc_gen_er(int scale, uint32_t d, uint64_t seed, uint32_t* rows, uint32_t* cols) {
    const uint32_t n = 1u << scale;
    for (uint32_t j = 0; j < n; ++j) {
        uint64_t st = orc_split_seed(seed, j);
        uint32_t* col = rows + (uint64_t)j * d;
        uint32_t filled = 0;
        for (uint32_t t = n - d; t < n; ++t) {
            uint32_t r = (uint32_t)sm_below(&st, (uint64_t)t + 1);
            int seen = 0;
            for (uint32_t s = 0; s < filled; ++s)
                if (col[s] == r) { seen = 1; break; }
            col[filled] = seen ? t : r;
            cols[(uint64_t)j * d + filled] = j;
            ++filled;
        }
    }
}

/* gen_rmat draws (src/generate.cpp:56-81), before the dedup of :83-88 which
 * the caller performs (sort + unique). */
void orc_gen_rmat_draws(int scale, uint32_t ef, uint64_t seed, double a, double b, double c,
                        uint32_t* rows, uint32_t* cols) {
    const uint64_t nedges = (uint64_t)ef << scale;
    const double cut_a = a, cut_ab = a + b, cut_abc = a + b + c;
    for (uint64_t e = 0; e < nedges; ++e) {
        uint64_t st = orc_split_seed(seed, e);
        uint32_t row = 0, col = 0;
        for (int level = scale - 1; level >= 0; --level) {
            double u = sm_unit(&st);
            if (u >= cut_ab) row |= 1u << level;
            if (u >= cut_abc || (u >= cut_a && u < cut_ab)) col |= 1u << level;
        }
        rows[e] = row;
        cols[e] = col;
    }
}

/* ---------------- choose_nbins (src/pb_spgemm.cpp:10-18) ---------------- */
static uint64_t bit_ceil64(uint64_t x) {
    uint64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}
static int ceil_log2_64(uint64_t x) { /* include/spgemm/pb_spgemm.hpp:20 */
    if (x <= 1) return 0;
    int b = 0;
    x -= 1;
    while (x) { ++b; x >>= 1; }
    return b;
}
uint32_t orc_choose_nbins(uint64_t flop, uint32_t nrows, uint64_t l2_bytes, uint32_t tuple_bytes) {
    const uint64_t budget = l2_bytes / 2 > 1 ? l2_bytes / 2 : 1;
    const uint64_t raw = (flop * tuple_bytes + budget - 1) / budget;
    uint64_t n = bit_ceil64(raw > 1 ? raw : 1);
    if (n < 64) n = 64;
    if (n > 8192) n = 8192;
    while (n > nrows) n >>= 1;
    return (uint32_t)(n > 1 ? n : 1);
}

/* ---------------- the pipeline --------------------------------------- */
typedef struct {
    /* symbolic (pb_spgemm.cpp:86-139) */
    uint64_t flop;
    uint64_t* per_column_flop; /* [k] */
    uint32_t nbins;
    uint64_t* per_bin_flop;    /* [nbins] */
    uint32_t* bin_row_starts;  /* [nbins+1] */
    uint32_t uniform_rows_per_bin;
    /* counters (acceptance.cpp:46-58) */
    uint64_t tuples_into_sort;
    uint64_t merged_total;
    /* C in CSR */
    uint32_t m, n;
    uint64_t nnz;
    uint64_t* rowptr;
    uint32_t* colids;
    double* values;
} orc_result;

enum { ORC_OK = 0, ORC_PARAM = 1, ORC_INTERNAL = 2, ORC_NOMEM = 3 };

/* insertion_sort_records (pb_spgemm.hpp:121-133) */
static void ins_sort(uint64_t* k, double* v, size_t n) {
    for (size_t i = 1; i < n; ++i) {
        uint64_t kk = k[i];
        double vv = v[i];
        size_t j = i;
        for (; j > 0 && k[j - 1] > kk; --j) { k[j] = k[j - 1]; v[j] = v[j - 1]; }
        k[j] = kk;
        v[j] = vv;
    }
}

/* detail::radix_pass, American-flag MSD on 8-bit digits (pb_spgemm.hpp:139-175) */
static void radix_pass(uint64_t* keys, double* vals, size_t n, const int* shifts, int nlevels,
                       int level) {
    if (n < 32) { ins_sort(keys, vals, n); return; }
    if (level >= nlevels) return;
    const int shift = shifts[level];
    size_t count[256] = {0}, start[257], next[256];
    for (size_t i = 0; i < n; ++i) ++count[(keys[i] >> shift) & 0xFF];
    start[0] = 0;
    for (int b = 0; b < 256; ++b) start[b + 1] = start[b] + count[b];
    memcpy(next, start, sizeof next);
    for (int b = 0; b < 256; ++b) {
        while (next[b] < start[b + 1]) {
            const size_t at = next[b];
            const int t = (int)((keys[at] >> shift) & 0xFF);
            if (t == b) {
                ++next[b];
            } else {
                uint64_t tk = keys[at]; keys[at] = keys[next[t]]; keys[next[t]] = tk;
                double tv = vals[at]; vals[at] = vals[next[t]]; vals[next[t]] = tv;
                ++next[t];
            }
        }
    }
    for (int b = 0; b < 256; ++b)
        if (count[b] > 1) radix_pass(keys + start[b], vals + start[b], count[b], shifts, nlevels, level + 1);
}

/* sort_bin_records (pb_spgemm.hpp:181-197): skip bytes constant in the run */
static void sort_bin(uint64_t* keys, double* vals, size_t n, int key_bytes) {
    if (n < 2) return;
    if (n < 32) { ins_sort(keys, vals, n); return; }
    uint64_t diff = 0;
    for (size_t i = 1; i < n; ++i) diff |= keys[i] ^ keys[0];
    if (!diff) return;
    int shifts[8], nlevels = 0;
    for (int byte = key_bytes - 1; byte >= 0; --byte)
        if ((diff >> (8 * byte)) & 0xFF) shifts[nlevels++] = 8 * byte;
    radix_pass(keys, vals, n, shifts, nlevels, 0);
}

/* compress_bin_records, two-pointer merge (pb_spgemm.hpp:202-216) */
static size_t compress_bin(uint64_t* keys, double* vals, size_t n) {
    if (!n) return 0;
    size_t w = 0;
    for (size_t r = 1; r < n; ++r) {
        if (keys[r] == keys[w]) vals[w] += vals[r];
        else { ++w; keys[w] = keys[r]; vals[w] = vals[r]; }
    }
    return w + 1;
}

void orc_free(orc_result* r) {
    if (!r) return;
    free(r->per_column_flop); free(r->per_bin_flop); free(r->bin_row_starts);
    free(r->rowptr); free(r->colids); free(r->values);
    free(r);
}

/*
 * pb_multiply (pb_spgemm.cpp:330-361): symbolic -> make_bins -> expand ->
 * sort_bins -> compress_bins -> convert_csr. Single-threaded: expand appends
 * straight into the bins in (k, p, q) order, which is the order the
 * reference's expand produces with one thread once its local-bin flushes are
 * drained (pb_spgemm.cpp:216-238).
 */
int orc_pb_multiply(uint32_t m, uint32_t k, uint64_t annz, const uint64_t* a_colptr,
                    const uint32_t* a_rowids, const double* a_vals, uint32_t bk, uint32_t n,
                    uint64_t bnnz, const uint64_t* b_rowptr, const uint32_t* b_colids,
                    const double* b_vals, uint32_t cfg_nbins, uint32_t lbin_bytes,
                    uint64_t l2_bytes, int balanced, orc_result** out) {
    (void)annz; (void)bnnz;
    *out = NULL;
    if (k != bk) return ORC_PARAM;                                    /* types.hpp:97-102 */
    if (cfg_nbins && (cfg_nbins & (cfg_nbins - 1))) return ORC_PARAM; /* pb_spgemm.cpp:88 */
    orc_result* r = (orc_result*)calloc(1, sizeof *r);
    if (!r) return ORC_NOMEM;
    r->m = m; r->n = n;

    /* per-column flop + overflow-checked total (pb_spgemm.cpp:97-105) */
    r->per_column_flop = (uint64_t*)malloc(sizeof(uint64_t) * (k ? k : 1));
    for (uint32_t i = 0; i < k; ++i) {
        r->per_column_flop[i] = (a_colptr[i + 1] - a_colptr[i]) * (b_rowptr[i + 1] - b_rowptr[i]);
        if (__builtin_add_overflow(r->flop, r->per_column_flop[i], &r->flop)) {
            orc_free(r);
            return ORC_PARAM;
        }
    }
    /* bin count and uniform starts (pb_spgemm.cpp:109-120) */
    const int col_bits = ceil_log2_64(n);
    uint32_t nbins = cfg_nbins ? cfg_nbins : orc_choose_nbins(r->flop, m, l2_bytes, 12);
    uint32_t rpb = (uint32_t)(((uint64_t)m + nbins - 1) / nbins);
    if (!cfg_nbins && ceil_log2_64(rpb) + col_bits > 32) {
        nbins = orc_choose_nbins(r->flop, m, l2_bytes, 16);
        rpb = (uint32_t)(((uint64_t)m + nbins - 1) / nbins);
    }
    r->nbins = nbins;
    r->uniform_rows_per_bin = rpb;
    r->bin_row_starts = (uint32_t*)malloc(sizeof(uint32_t) * (nbins + 1));
    for (uint32_t b = 0; b <= nbins; ++b) {
        uint64_t s = (uint64_t)b * rpb;
        r->bin_row_starts[b] = (uint32_t)(s < m ? s : m);
    }
    uint32_t* row_bin = (uint32_t*)malloc(sizeof(uint32_t) * (m ? m : 1));
    for (uint32_t row = 0; row < m; ++row) row_bin[row] = rpb ? row / rpb : 0;
    /* bin_flop (pb_spgemm.cpp:36-54) */
    r->per_bin_flop = (uint64_t*)calloc(nbins, sizeof(uint64_t));
    for (uint32_t i = 0; i < k; ++i) {
        const uint64_t bn = b_rowptr[i + 1] - b_rowptr[i];
        for (uint64_t p = a_colptr[i]; p < a_colptr[i + 1]; ++p) r->per_bin_flop[row_bin[a_rowids[p]]] += bn;
    }
    /* balanced_starts (pb_spgemm.cpp:58-82, 122-137) */
    if (balanced) {
        uint64_t maxb = 0;
        for (uint32_t b = 0; b < nbins; ++b) if (r->per_bin_flop[b] > maxb) maxb = r->per_bin_flop[b];
        const uint32_t tb = ceil_log2_64(rpb) + col_bits <= 32 ? 12 : 16;
        if (maxb * tb > l2_bytes) {
            uint64_t* row_flop = (uint64_t*)calloc(m ? m : 1, sizeof(uint64_t));
            for (uint32_t i = 0; i < k; ++i) {
                const uint64_t bn = b_rowptr[i + 1] - b_rowptr[i];
                for (uint64_t p = a_colptr[i]; p < a_colptr[i + 1]; ++p) row_flop[a_rowids[p]] += bn;
            }
            for (uint32_t b = 0; b <= nbins; ++b) r->bin_row_starts[b] = m;
            r->bin_row_starts[0] = 0;
            const double target = (double)r->flop / nbins;
            uint64_t acc = 0;
            uint32_t bin = 1;
            for (uint32_t row = 0; row < m && bin < nbins; ++row) {
                acc += row_flop[row];
                if ((double)acc >= target * bin) r->bin_row_starts[bin++] = row + 1;
            }
            free(row_flop);
            r->uniform_rows_per_bin = 0;
            for (uint32_t b = 0; b < nbins; ++b)
                for (uint32_t row = r->bin_row_starts[b]; row < r->bin_row_starts[b + 1]; ++row) row_bin[row] = b;
            memset(r->per_bin_flop, 0, sizeof(uint64_t) * nbins);
            for (uint32_t i = 0; i < k; ++i) {
                const uint64_t bn = b_rowptr[i + 1] - b_rowptr[i];
                for (uint64_t p = a_colptr[i]; p < a_colptr[i + 1]; ++p) r->per_bin_flop[row_bin[a_rowids[p]]] += bn;
            }
        }
    }
    /* expand's lbin_bytes check (pb_spgemm.cpp:252-253) */
    if (lbin_bytes == 0 || lbin_bytes % 16 != 0) {
        free(row_bin);
        orc_free(r);
        return ORC_PARAM;
    }
    /* make_bins (pb_spgemm.cpp:141-176) */
    uint32_t max_span = 0;
    for (uint32_t b = 0; b < nbins; ++b) {
        uint32_t s = r->bin_row_starts[b + 1] - r->bin_row_starts[b];
        if (s > max_span) max_span = s;
    }
    const int key_bytes = ceil_log2_64(max_span) + col_bits <= 32 ? 4 : 8;
    uint64_t* offsets = (uint64_t*)malloc(sizeof(uint64_t) * (nbins + 1));
    uint64_t* fill = (uint64_t*)calloc(nbins, sizeof(uint64_t));
    uint64_t* merged = (uint64_t*)calloc(nbins, sizeof(uint64_t));
    offsets[0] = 0;
    for (uint32_t b = 0; b < nbins; ++b) offsets[b + 1] = offsets[b] + r->per_bin_flop[b];
    const uint64_t total = offsets[nbins];
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (total ? total : 1));
    double* vals = (double*)malloc(sizeof(double) * (total ? total : 1));
    if (!keys || !vals) {
        free(row_bin); free(offsets); free(fill); free(merged); free(keys); free(vals);
        orc_free(r);
        return ORC_NOMEM;
    }
    /* expand (pb_spgemm.cpp:216-234): key = (row - bin_base) << col_bits | col */
    for (uint32_t i = 0; i < k; ++i) {
        const uint64_t blo = b_rowptr[i], bhi = b_rowptr[i + 1];
        if (blo == bhi) continue;
        for (uint64_t p = a_colptr[i]; p < a_colptr[i + 1]; ++p) {
            const uint32_t row = a_rowids[p];
            const double av = a_vals[p];
            const uint32_t bin = row_bin[row];
            const uint64_t row_part = (uint64_t)(row - r->bin_row_starts[bin]) << col_bits;
            for (uint64_t q = blo; q < bhi; ++q) {
                const uint64_t at = offsets[bin] + fill[bin]++;
                keys[at] = row_part | b_colids[q];
                vals[at] = av * b_vals[q];
            }
        }
    }
    int rc = ORC_OK;
    for (uint32_t b = 0; b < nbins; ++b) {
        r->tuples_into_sort += fill[b];
        if (fill[b] != offsets[b + 1] - offsets[b]) rc = ORC_INTERNAL; /* :241-245 */
    }
    if (r->tuples_into_sort != r->flop) rc = ORC_INTERNAL; /* :342-345 */
    /* sort_bins + compress_bins (pb_spgemm.cpp:260-284) */
    for (uint32_t b = 0; b < nbins && rc == ORC_OK; ++b) {
        sort_bin(keys + offsets[b], vals + offsets[b], fill[b], key_bytes);
        merged[b] = compress_bin(keys + offsets[b], vals + offsets[b], fill[b]);
        r->merged_total += merged[b];
    }
    /* convert_csr (pb_spgemm.cpp:288-321) */
    if (rc == ORC_OK) {
        r->rowptr = (uint64_t*)calloc((uint64_t)m + 1, sizeof(uint64_t));
        const uint64_t mask = col_bits >= 64 ? ~0ULL : ((1ULL << col_bits) - 1);
        for (uint32_t b = 0; b < nbins; ++b)
            for (uint64_t p = offsets[b]; p < offsets[b] + merged[b]; ++p)
                ++r->rowptr[r->bin_row_starts[b] + (keys[p] >> col_bits) + 1];
        for (uint32_t row = 0; row < m; ++row) r->rowptr[row + 1] += r->rowptr[row];
        r->nnz = r->rowptr[m];
        r->colids = (uint32_t*)malloc(sizeof(uint32_t) * (r->nnz ? r->nnz : 1));
        r->values = (double*)malloc(sizeof(double) * (r->nnz ? r->nnz : 1));
        for (uint32_t b = 0; b < nbins; ++b) {
            uint64_t at = r->rowptr[r->bin_row_starts[b]];
            for (uint64_t p = offsets[b]; p < offsets[b] + merged[b]; ++p, ++at) {
                r->colids[at] = (uint32_t)(keys[p] & mask);
                r->values[at] = vals[p];
            }
        }
        if (r->nnz != r->merged_total) rc = ORC_INTERNAL; /* :358-359 */
    }
    free(row_bin); free(offsets); free(fill); free(merged); free(keys); free(vals);
    if (rc != ORC_OK) { orc_free(r); return rc; }
    *out = r;
    return ORC_OK;
}

/* accessors for ctypes */
uint64_t orc_res_nnz(const orc_result* r) { return r->nnz; }
uint32_t orc_res_nbins(const orc_result* r) { return r->nbins; }
void orc_res_get(const orc_result* r, uint64_t* rowptr, uint32_t* colids, double* vals) {
    memcpy(rowptr, r->rowptr, sizeof(uint64_t) * ((uint64_t)r->m + 1));
    memcpy(colids, r->colids, sizeof(uint32_t) * r->nnz);
    memcpy(vals, r->values, sizeof(double) * r->nnz);
}
void orc_res_counters(const orc_result* r, uint64_t* c) {
    c[0] = r->flop; c[1] = r->tuples_into_sort; c[2] = r->merged_total; c[3] = r->uniform_rows_per_bin;
}
void orc_res_symbolic(const orc_result* r, uint64_t* per_column_flop, uint32_t k, uint64_t* per_bin_flop,
                      uint32_t* bin_row_starts) {
    memcpy(per_column_flop, r->per_column_flop, sizeof(uint64_t) * k);
    memcpy(per_bin_flop, r->per_bin_flop, sizeof(uint64_t) * r->nbins);
    memcpy(bin_row_starts, r->bin_row_starts, sizeof(uint32_t) * (r->nbins + 1));
}
