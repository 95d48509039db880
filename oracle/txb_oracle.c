/*
 * txb_oracle.c — CPU restatement of the reference element-integration path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library, and only as the checker
 * (or the timed CPU baseline) — never as the thing measured or shipped.  The
 * product path (paper_1607_04245_b200/) never links or calls it.
 *
 * What it restates (pinned per-cell operation order, reference.py:10-19):
 *
 *   for each quadrature point q (ascending):
 *       T[q][b][k]  = sum_j D[q][b][j] * invJ[j][k]           (j ascending, from 0)
 *       u[c]        = sum_b coeff[b][c] * B[q][b]               (b ascending, from 0)
 *       grad[c][k]  = sum_b coeff[b][c] * T[q][b][k]            (b ascending, from 0)
 *       a0          = aux_const[cell]            (P0)           (_kernels_cy.pyx:89-94)
 *                   = sum_b aux_nodal[cell][b] * B[q][b]  (P1)
 *       f1 by form: 0 copy, 1 a0*grad, 2 0.5*(grad[c][k]+grad[k][c])   (pyx:98-108,
 *                   physics.py:171-257)
 *       f1s[q][c][k] = (f1[k] * detJ) * w[q]                    (pyx:109-111)
 *   for each (b, c):  e = 0;  for q, k:  e += T[q][b][k] * f1s[q][c][k]
 *                                                               (pyx:113-123)
 *
 * Compiled with -ffp-contract=off (as the reference lane, pkg/setup.py:17-20)
 * so every multiply and add rounds separately: the f64 entry point is
 * bit-identical to txfem.reference.integrate_reference and the f32 entry
 * point to the reference's compiled lane on f32 inputs.  Both claims are
 * checked against tests/golden/ (generated from the reference itself).
 *
 * Layouts (C-contiguous, one dtype), as _kernels_cy.pyx:40-48:
 *   basis (n_q, n_b), basis_der (n_q, n_b, d), weights (n_q),
 *   inv_j (n, d, d) row-major, det_j (n), coeffs (n, n_b, n_comp),
 *   aux (n, 1) for aux_mode 1 / (n, n_b, 1) for aux_mode 2 / NULL,
 *   out (n, n_b, n_comp) fully overwritten.
 */
#include <stdint.h>
#include <stddef.h>

#define MAX_D 3
#define MAX_B 4
#define MAX_COMP 3
#define MAX_Q 8

#define DEFINE_ORACLE(NAME, real)                                                   \
int NAME(int form_code, int aux_mode, int d, int n_b, int n_q, int n_comp,          \
         int64_t n, const real* basis, const real* basis_der, const real* weights,  \
         const real* inv_j, const real* det_j, const real* coeffs, const real* aux, \
         real* out)                                                                 \
{                                                                                   \
    if (d > MAX_D || n_b > MAX_B || n_comp > MAX_COMP || n_q > MAX_Q) return -1;   \
    if (form_code < 0 || form_code > 2 || aux_mode < 0 || aux_mode > 2) return -1;  \
    for (int64_t cell = 0; cell < n; ++cell) {                                      \
        const real* J = inv_j + cell * d * d;                                       \
        const real* C = coeffs + cell * n_b * n_comp;                               \
        real trans[MAX_Q][MAX_B][MAX_D];                                            \
        real f1s[MAX_Q][MAX_COMP][MAX_D];                                           \
        /* quadrature phase */                                                      \
        for (int q = 0; q < n_q; ++q) {                                             \
            for (int b = 0; b < n_b; ++b)                                           \
                for (int k = 0; k < d; ++k) {                                       \
                    real acc = 0;                                                   \
                    for (int j = 0; j < d; ++j)                                     \
                        acc = acc + basis_der[(q * n_b + b) * d + j] * J[j * d + k];\
                    trans[q][b][k] = acc;                                           \
                }                                                                   \
            real u[MAX_COMP], grad[MAX_COMP][MAX_D];                                \
            for (int c = 0; c < n_comp; ++c) {                                      \
                u[c] = 0;                                                           \
                for (int k = 0; k < d; ++k) grad[c][k] = 0;                         \
            }                                                                       \
            for (int b = 0; b < n_b; ++b)                                           \
                for (int c = 0; c < n_comp; ++c) {                                  \
                    u[c] = u[c] + C[b * n_comp + c] * basis[q * n_b + b];           \
                    for (int k = 0; k < d; ++k)                                     \
                        grad[c][k] = grad[c][k] + C[b * n_comp + c] * trans[q][b][k];\
                }                                                                   \
            (void)u;                                                                \
            real a0 = 0;                                                            \
            if (aux_mode == 1) a0 = aux[cell];                                      \
            else if (aux_mode == 2)                                                 \
                for (int b = 0; b < n_b; ++b)                                       \
                    a0 = a0 + aux[cell * n_b + b] * basis[q * n_b + b];             \
            const real det = det_j[cell], wq = weights[q];                          \
            for (int c = 0; c < n_comp; ++c) {                                      \
                real fv[MAX_D];                                                     \
                for (int k = 0; k < d; ++k) {                                       \
                    if (form_code == 0) fv[k] = grad[c][k];                         \
                    else if (form_code == 1) fv[k] = a0 * grad[c][k];               \
                    else { real t = grad[c][k] + grad[k][c]; fv[k] = (real)0.5 * t; }\
                }                                                                   \
                for (int k = 0; k < d; ++k) {                                       \
                    real tmp = fv[k] * det;                                         \
                    f1s[q][c][k] = tmp * wq;                                        \
                }                                                                   \
            }                                                                       \
        }                                                                           \
        /* basis phase */                                                           \
        for (int b = 0; b < n_b; ++b)                                               \
            for (int c = 0; c < n_comp; ++c) {                                      \
                real e = 0;                                                         \
                for (int q = 0; q < n_q; ++q)                                       \
                    for (int k = 0; k < d; ++k) {                                   \
                        real acc = 0;                                               \
                        for (int j = 0; j < d; ++j)                                 \
                            acc = acc + basis_der[(q * n_b + b) * d + j] * J[j * d + k];\
                        e = e + acc * f1s[q][c][k];                                 \
                    }                                                               \
                out[(cell * n_b + b) * n_comp + c] = e;                             \
            }                                                                       \
    }                                                                               \
    return 0;                                                                       \
}

DEFINE_ORACLE(txb_oracle_integrate_f64, double)
DEFINE_ORACLE(txb_oracle_integrate_f32, float)

/* Gather per-cell coefficient blocks from an interleaved global vector
 * (mesh.gather_coefficients, mesh.py:202-217): out[c][b][k] = g[cells[c][b]*n_comp+k]. */
void txb_oracle_gather_f64(int64_t n, int n_b, int n_comp, const int64_t* cells,
                           const double* global, double* out)
{
    for (int64_t c = 0; c < n; ++c)
        for (int b = 0; b < n_b; ++b)
            for (int k = 0; k < n_comp; ++k)
                out[(c * n_b + b) * n_comp + k] = global[cells[c * n_b + b] * n_comp + k];
}

/* Scatter-add element vectors in ascending (cell, b) order
 * (mesh.scatter_add_element_vectors / np.add.at, mesh.py:220-234). */
#define DEFINE_SCATTER(NAME, real)                                                  \
void NAME(int64_t n, int n_b, int n_comp, int64_t n_vertices, const int64_t* cells, \
          const real* elem, real* out)                                              \
{                                                                                   \
    for (int64_t v = 0; v < n_vertices * n_comp; ++v) out[v] = 0;                   \
    for (int64_t c = 0; c < n; ++c)                                                 \
        for (int b = 0; b < n_b; ++b)                                               \
            for (int k = 0; k < n_comp; ++k) {                                      \
                int64_t g = cells[c * n_b + b] * n_comp + k;                        \
                out[g] = out[g] + elem[(c * n_b + b) * n_comp + k];                 \
            }                                                                       \
}
DEFINE_SCATTER(txb_oracle_scatter_add_f64, double)
DEFINE_SCATTER(txb_oracle_scatter_add_f32, float)
