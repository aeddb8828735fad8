/*
 * tk_oracle.c -- CPU restatement of the reference kernels, used ONLY as a test
 * checker and as the CPU-baseline leg of bench.py.  Never linked into, loaded
 * by, or called from the product path (paper_2510_01495_b200/).
 *
 * Restates pkg/src/tenkern/_ckernels.pyx of the reference (arXiv 2510.01495
 * companion package "tenkern"):
 *   - dot            : _dot_impl          _ckernels.pyx:40-45
 *   - matvec         : _matvec_impl       _ckernels.pyx:48-56
 *   - ttv pipeline   : _ttv_pipeline      _ckernels.pyx:313-367
 *        scale/project  _scale_project    _ckernels.pyx:129-150
 *        argsort        _argsort_rows     _ckernels.pyx:229-259
 *                       _counting_passes  _ckernels.pyx:202-226
 *                       _merge_argsort    _ckernels.pyx:164-199
 *        group-sum      _group_sum_nonzero _ckernels.pyx:262-295
 *
 * Arithmetic contract (what makes the GPU parity bit-exact): every product is
 * one IEEE binary64 multiply rounded to nearest, every sum a left-to-right
 * chain of binary64 adds rounded to nearest, no fused multiply-add (the
 * reference is built with -O3 and no -ffast-math / -march, pkg/setup.py:4-13).
 * This file is compiled with -ffp-contract=off for the same reason.
 *
 * Pinning: tests/test_oracle.py checks this restatement against the golden
 * vectors in tests/golden/ that tests/golden/make_golden.py produced by
 * running the reference itself (and, when oracle/_ref is built, against the
 * reference's compiled extension directly).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TKO_OK 0
#define TKO_EINDEX 4 /* mode-k index outside x: DimensionError in the reference */
#define TKO_ENOMEM 9

/* _ckernels.pyx:40-45 -- one accumulator, starts at 0.0, index order. */
double tko_dot(const double *x, const double *y, int64_t n) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += x[i] * y[i];
    return acc;
}

/* _ckernels.pyx:48-56 -- row loop outer, each row reduced exactly like dot. */
void tko_matvec(const double *a, int64_t rows, int64_t cols, const double *x, double *y) {
    for (int64_t i = 0; i < rows; ++i) {
        const double *row = a + i * cols;
        double acc = 0.0;
        for (int64_t j = 0; j < cols; ++j) acc += row[j] * x[j];
        y[i] = acc;
    }
}

/* lexicographic row <= (stable merge predicate), _ckernels.pyx:153-161 */
static int row_le(const int64_t *proj, int64_t dk, int64_t ra, int64_t rb) {
    const int64_t *a = proj + ra * dk, *b = proj + rb * dk;
    for (int64_t c = 0; c < dk; ++c) {
        if (a[c] < b[c]) return 1;
        if (a[c] > b[c]) return 0;
    }
    return 1;
}

/* bottom-up stable merge sort of order[] by projected rows, _ckernels.pyx:164-199 */
static void merge_argsort(const int64_t *proj, int64_t dk, int64_t n, int64_t *order, int64_t *buf) {
    for (int64_t width = 1; width < n; width *= 2) {
        for (int64_t lo = 0; lo + width < n; lo += 2 * width) {
            int64_t mid = lo + width, hi = lo + 2 * width < n ? lo + 2 * width : n;
            int64_t a = lo, b = mid, i = lo;
            while (a < mid && b < hi) buf[i++] = row_le(proj, dk, order[a], order[b]) ? order[a++] : order[b++];
            while (a < mid) buf[i++] = order[a++];
            while (b < hi) buf[i++] = order[b++];
            memcpy(order + lo, buf + lo, (size_t)(hi - lo) * sizeof(int64_t));
        }
    }
}

/* LSD counting sort, last projected column first, _ckernels.pyx:202-226 */
static void counting_passes(const int64_t *proj, int64_t dk, int64_t n, const int64_t *dims,
                            int64_t *order, int64_t *scratch, int64_t *counts) {
    for (int64_t col = dk - 1; col >= 0; --col) {
        int64_t nb = dims[col], total = 0;
        memset(counts, 0, (size_t)nb * sizeof(int64_t));
        for (int64_t i = 0; i < n; ++i) counts[proj[order[i] * dk + col]]++;
        for (int64_t i = 0; i < nb; ++i) { int64_t c = counts[i]; counts[i] = total; total += c; }
        for (int64_t i = 0; i < n; ++i) {
            int64_t key = proj[order[i] * dk + col];
            scratch[counts[key]++] = order[i];
        }
        memcpy(order, scratch, (size_t)n * sizeof(int64_t));
    }
}

/*
 * Mode-k TTV over row-major (nnz, d) subs.  Output capacity: nnz rows.
 * Returns TKO_OK and *out_u, or TKO_EINDEX (no outputs written).
 * Structural guards (d >= 2, 0 <= k < d, nx == shape[k]) are the caller's
 * (oracle.py), mirroring _check_ttv, _ckernels.pyx:298-310.
 */
int tko_ttv(int32_t d, const int64_t *shape, int64_t nnz, const int64_t *subs, const double *vals,
            const double *x, int64_t nx, int32_t k, int64_t *out_subs, double *out_vals, int64_t *out_u) {
    const int64_t dk = d - 1;
    *out_u = 0;
    if (nnz == 0) return TKO_OK; /* _ckernels.pyx:322-327 */

    int64_t dims[64];
    int64_t max_dim = 0;
    for (int32_t m = 0, c = 0; m < d; ++m)
        if (m != k) { dims[c] = shape[m]; if (shape[m] > max_dim) max_dim = shape[m]; ++c; }
    /* counting sort planned when max_dim <= max(65536, 4 nnz), _ckernels.pyx:334-336 */
    int64_t cap = 4 * nnz > 65536 ? 4 * nnz : 65536;
    int counting = max_dim <= cap;

    double *w = malloc((size_t)nnz * sizeof(double));
    int64_t *proj = malloc((size_t)(nnz * (dk ? dk : 1)) * sizeof(int64_t));
    int64_t *order = malloc((size_t)nnz * sizeof(int64_t));
    int64_t *scratch = malloc((size_t)nnz * sizeof(int64_t));
    int64_t *counts = counting ? malloc((size_t)(max_dim ? max_dim : 1) * sizeof(int64_t)) : NULL;
    if (!w || !proj || !order || !scratch || (counting && !counts)) {
        free(w); free(proj); free(order); free(scratch); free(counts);
        return TKO_ENOMEM;
    }

    /* scale + project with the mode-k bound checked in the same pass, _ckernels.pyx:129-150 */
    for (int64_t r = 0; r < nnz; ++r) {
        int64_t idx = subs[r * d + k];
        if (idx < 0 || idx >= nx) {
            free(w); free(proj); free(order); free(scratch); free(counts);
            return TKO_EINDEX;
        }
        w[r] = vals[r] * x[idx];
        for (int32_t m = 0, c = 0; m < d; ++m)
            if (m != k) proj[r * dk + c++] = subs[r * d + m];
    }

    /* stable argsort of projected rows, _ckernels.pyx:229-259 */
    for (int64_t i = 0; i < nnz; ++i) order[i] = i;
    if (nnz > 1 && dk > 0) {
        if (counting) {
            for (int64_t c = 0; c < dk && counting; ++c) {
                if (dims[c] > max_dim) { counting = 0; break; }
                for (int64_t i = 0; i < nnz; ++i) {
                    int64_t v = proj[i * dk + c];
                    if (v < 0 || v >= dims[c]) { counting = 0; break; }
                }
            }
        }
        if (counting) counting_passes(proj, dk, nnz, dims, order, scratch, counts);
        else merge_argsort(proj, dk, nnz, order, scratch);
    }

    /* run-length group sum in original-row order, drop exact zeros, _ckernels.pyx:262-295 */
    int64_t u = 0;
    for (int64_t i = 0; i < nnz;) {
        int64_t ra = order[i];
        double acc = w[ra];
        int64_t j = i + 1;
        for (; j < nnz; ++j) {
            int64_t rb = order[j];
            if (memcmp(proj + ra * dk, proj + rb * dk, (size_t)dk * sizeof(int64_t)) != 0) break;
            acc += w[rb];
        }
        if (acc != 0.0) {
            memcpy(out_subs + u * dk, proj + ra * dk, (size_t)dk * sizeof(int64_t));
            out_vals[u++] = acc;
        }
        i = j;
    }
    *out_u = u;
    free(w); free(proj); free(order); free(scratch); free(counts);
    return TKO_OK;
}
