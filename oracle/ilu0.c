/*
 * TEST INFRASTRUCTURE ONLY — never linked into the product library.
 *
 * Plain-C restatement of the reference's numba ILU(0) kernels, used as the
 * CPU oracle (and as the CPU baseline in bench.py) for parity checks:
 *   oracle_ilu0_factor  <-  paradiff/linalg.py:63-97   (_ilu0_factor)
 *   oracle_ilu0_solve   <-  paradiff/linalg.py:100-113  (_ilu0_solve)
 *
 * CSR must have sorted column indices (linalg.py:47-52).  The factor works in
 * place: unit-lower L strictly below the diagonal, U on and above, both on
 * the original pattern.  Built with -ffp-contract=off so products and
 * differences round separately, as numba/LLVM does by default.
 */
#include <stdint.h>
#include <stdlib.h>

/* Returns -1 on success, otherwise the row whose pivot is zero/missing
 * (first failing row in natural order, like linalg.py:85-94). */
int64_t oracle_ilu0_factor(int64_t n, const int64_t *rowptr, const int64_t *col,
                           double *val, int64_t *diag)
{
    int64_t *where = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    if (!where) return -2;
    for (int64_t i = 0; i < n; ++i) where[i] = -1;
    int64_t bad = -1;
    for (int64_t i = 0; i < n && bad < 0; ++i) {
        const int64_t a = rowptr[i], e = rowptr[i + 1];
        diag[i] = -1;
        for (int64_t p = a; p < e; ++p) {
            where[col[p]] = p;
            if (col[p] == i) diag[i] = p;
        }
        for (int64_t pk = a; pk < e; ++pk) {
            const int64_t k = col[pk];
            if (k >= i) break;
            const int64_t dk = diag[k];
            const double piv = val[dk];
            if (piv == 0.0) { bad = k; break; }
            const double lik = val[pk] / piv;
            val[pk] = lik;
            for (int64_t p = dk + 1; p < rowptr[k + 1]; ++p) {
                const int64_t q = where[col[p]];
                if (q >= 0) {
                    const double prod = lik * val[p];
                    val[q] = val[q] - prod;
                }
            }
        }
        if (bad < 0 && (diag[i] < 0 || val[diag[i]] == 0.0)) bad = i;
        for (int64_t p = a; p < e; ++p) where[col[p]] = -1;
    }
    free(where);
    return bad;
}

void oracle_ilu0_solve(int64_t n, const int64_t *rowptr, const int64_t *col,
                       const double *val, const int64_t *diag,
                       const double *b, double *x)
{
    for (int64_t i = 0; i < n; ++i) {           /* unit lower */
        double s = b[i];
        for (int64_t p = rowptr[i]; p < diag[i]; ++p) {
            const double prod = val[p] * x[col[p]];
            s = s - prod;
        }
        x[i] = s;
    }
    for (int64_t i = n - 1; i >= 0; --i) {      /* upper */
        double s = x[i];
        for (int64_t p = diag[i] + 1; p < rowptr[i + 1]; ++p) {
            const double prod = val[p] * x[col[p]];
            s = s - prod;
        }
        x[i] = s / val[diag[i]];
    }
}
