"""User physics forms for the run-time compiled lane's parity tests — TEST
INFRASTRUCTURE ONLY (imported by tests/ and tests/golden/make_golden.py).

Each spec is the same form written twice, the way the reference expects a
user to write one (txfem/physics.py:260-304, tests/conftest.py:43-79):
  * source text in the string-injection dialect (what the CUDA lane compiles);
  * numpy ``f1_many`` / ``f0_many`` evaluating the same expressions in the
    same order (what the reference's python lane, txfem/_kernels_py.py:53-65,
    calls).
Coverage beyond the shipped forms: an f0 term (reaction), several auxiliary
fields, P0 and P1 aux, the P1 aux gradient (uses_grad_a), vector-valued f0.
"""

from __future__ import annotations

import numpy as np

SIG = "(const real u[], const realv gradU[], const real a[], const realv gradA[], int comp)"
AX = "xyz"


def _reaction(dim):
    """tests/conftest.py:43-79: f0 = u, f1 = grad u."""

    def f1_many(u, grad_u, a, grad_a):
        return grad_u.copy()

    def f0_many(u, grad_u, a, grad_a):
        return u.copy()

    return dict(name="reaction", dim=dim, n_comp=1, n_aux=0, aux=None, uses_grad_a=False,
                source_f1=f"realv f1_reaction{SIG}\n{{\n  return gradU[comp];\n}}\n",
                source_f0=f"real f0_reaction{SIG}\n{{\n  return u[comp];\n}}\n",
                f1_many=f1_many, f0_many=f0_many, flops_f1=0, flops_f0=0)


def _advect(dim):
    """Two P1 auxiliary fields with their gradients: f1 = a0 grad u + u grad a1,
    f0 = a1 u + grad a0 . grad u."""

    def f1_many(u, grad_u, a, grad_a):
        return a[:, 0, None, None] * grad_u + u[:, :, None] * grad_a[:, None, 1, :]

    def f0_many(u, grad_u, a, grad_a):
        s = grad_a[:, 0, None, 0] * grad_u[:, :, 0]
        for k in range(1, grad_u.shape[-1]):
            s = s + grad_a[:, 0, None, k] * grad_u[:, :, k]
        return a[:, 1, None] * u + s

    return dict(name="advect", dim=dim, n_comp=1, n_aux=2, aux="p1", uses_grad_a=True,
                source_f1=f"realv f1_advect{SIG}\n{{\n  return a[0]*gradU[comp] + u[comp]*gradA[1];\n}}\n",
                source_f0=f"real f0_advect{SIG}\n{{\n  return a[1]*u[comp] + dot(gradA[0], gradU[comp]);\n}}\n",
                f1_many=f1_many, f0_many=f0_many, flops_f1=3 * dim, flops_f0=2 * dim + 1)


def _elastic_body(dim):
    """Vector-valued (n_comp = d) with one P0 field: f1 = a0 sym(grad u) row,
    f0 = a0 u (body-force-like)."""
    cases = []
    for c in range(dim):
        rows = "".join(f"    f1.{AX[k]} = a[0]*(0.5*(gradU[{c}].{AX[k]} + gradU[{k}].{AX[c]}));\n"
                       for k in range(dim))
        cases.append(f"  case {c}:\n{rows}    break;\n")
    src1 = f"realv f1_elastic_body{SIG}\n{{\n  realv f1;\n  switch (comp) {{\n{''.join(cases)}  }}\n  return f1;\n}}\n"

    def f1_many(u, grad_u, a, grad_a):
        out = np.empty_like(grad_u)
        half = grad_u.dtype.type(0.5)
        for c in range(grad_u.shape[-1]):
            for k in range(grad_u.shape[-1]):
                out[:, c, k] = a[:, 0] * (half * (grad_u[:, c, k] + grad_u[:, k, c]))
        return out

    def f0_many(u, grad_u, a, grad_a):
        return a[:, 0, None] * u

    return dict(name="elastic_body", dim=dim, n_comp=dim, n_aux=1, aux="p0", uses_grad_a=False,
                source_f1=src1, source_f0=f"real f0_elastic_body{SIG}\n{{\n  return a[0]*u[comp];\n}}\n",
                f1_many=f1_many, f0_many=f0_many, flops_f1=3 * dim, flops_f0=1)


def _three_fields(dim):
    """Three P0 fields, no f0: f1 = a2 (a0 grad u) - a1 grad u."""

    def f1_many(u, grad_u, a, grad_a):
        return a[:, 2, None, None] * (a[:, 0, None, None] * grad_u) - a[:, 1, None, None] * grad_u

    return dict(name="three_fields", dim=dim, n_comp=1, n_aux=3, aux="p0", uses_grad_a=False,
                source_f1=f"realv f1_three_fields{SIG}\n{{\n  return a[2]*(a[0]*gradU[comp]) - a[1]*gradU[comp];\n}}\n",
                source_f0=None, f1_many=f1_many, f0_many=None, flops_f1=3 * dim, flops_f0=0)


SPECS = {"reaction": _reaction, "advect": _advect, "elastic_body": _elastic_body, "three_fields": _three_fields}


def spec(name: str, dim: int) -> dict:
    return SPECS[name](dim)


def make_form(user_form, name: str, dim: int):
    """Build the form with a ``user_form`` constructor (the reference's or ours)."""
    s = spec(name, dim)

    def f1(state, comp):  # scalar evaluator through the vectorised one (API completeness)
        a = None if state.a is None else state.a[None]
        ga = None if state.grad_a is None else state.grad_a[None]
        return s["f1_many"](state.u[None], state.grad_u[None], a, ga)[0, comp]

    kw = dict(n_aux=s["n_aux"], f1_many=s["f1_many"], uses_grad_a=s["uses_grad_a"])
    if s["f0_many"] is not None:
        def f0(state, comp):
            a = None if state.a is None else state.a[None]
            ga = None if state.grad_a is None else state.grad_a[None]
            return s["f0_many"](state.u[None], state.grad_u[None], a, ga)[0, comp]

        kw.update(f0=f0, f0_many=s["f0_many"], flops_f0=s["flops_f0"], source_f0=s["source_f0"])
    return user_form(s["name"], dim, s["n_comp"], f1, s["flops_f1"], s["source_f1"], **kw)
