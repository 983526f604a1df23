/* Sequential lexicographic Gauss-Seidel sweeps over a CSR matrix.
 *
 * TEST INFRASTRUCTURE ONLY (oracle side).  Plain-C restatement of the
 * reference's numba loops `_gs_forward` / `_gs_backward`
 * (/root/reference/pkg/src/vtsopt/multigrid.py:35-64): for every row in
 * increasing (forward) or decreasing (backward) order,
 *     x[i] = (b[i] - sum_{j != i} a_ij x[j]) / a_ii,
 * accumulating the off-diagonal products in CSR storage order exactly as the
 * reference does.  Built by oracle/Makefile into oracle/_build/.
 */
#include <stdint.h>

void vts_oracle_gs_forward(const int64_t* indptr, const int64_t* indices, const double* data,
                           double* x, const double* b, int64_t n, int32_t sweeps) {
  for (int32_t s = 0; s < sweeps; ++s) {
    for (int64_t i = 0; i < n; ++i) {
      double acc = b[i];
      double diag = 0.0;
      for (int64_t jj = indptr[i]; jj < indptr[i + 1]; ++jj) {
        const int64_t j = indices[jj];
        if (j == i) diag = data[jj];
        else acc -= data[jj] * x[j];
      }
      x[i] = acc / diag;
    }
  }
}

void vts_oracle_gs_backward(const int64_t* indptr, const int64_t* indices, const double* data,
                            double* x, const double* b, int64_t n, int32_t sweeps) {
  for (int32_t s = 0; s < sweeps; ++s) {
    for (int64_t i = n - 1; i >= 0; --i) {
      double acc = b[i];
      double diag = 0.0;
      for (int64_t jj = indptr[i]; jj < indptr[i + 1]; ++jj) {
        const int64_t j = indices[jj];
        if (j == i) diag = data[jj];
        else acc -= data[jj] * x[j];
      }
      x[i] = acc / diag;
    }
  }
}
