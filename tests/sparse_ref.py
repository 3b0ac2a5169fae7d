"""Sparse-matrix reference of the Trotter energy (scipy), a third evaluator
beside the oracle's Pauli-string rotations and its JW-free determinant
evaluator: every generator is applied as exp(theta * A_g) |psi> with A_g the
sparse matrix of its JW image (scipy.sparse.linalg.expm_multiply: a Taylor /
Krylov matrix exponential, no closed-form rotation and no fused pattern logic),
and <psi|H|psi> term by term from the Pauli action on the index. Test
infrastructure only. Conventions: qubit 0 = least
significant bit; (P psi)[k] = i^ny (-1)^popc((k ^ x) & z) psi[k ^ x]."""
import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import expm_multiply

_IPOW = np.array([1, 1j, -1, -1j])


def _parity(v):
    return (np.bitwise_count(v) & 1).astype(np.int8)


def pauli_sparse(n, x, z):
    """CSR matrix of the string (x, z) with its i^ny phase (Hermitian)."""
    dim = 1 << n
    k = np.arange(dim, dtype=np.uint64)
    cols = k ^ np.uint64(x)
    ny = bin(int(x) & int(z)).count("1") & 3
    vals = _IPOW[ny] * (1.0 - 2.0 * _parity(cols & np.uint64(z)))
    return sp.csr_matrix((vals, (k.astype(np.int64), cols.astype(np.int64))), shape=(dim, dim))


def pauli_expect(n, psi, x, z):
    """<psi| P |psi> (complex) from the index action, O(2^n)."""
    dim = 1 << n
    k = np.arange(dim, dtype=np.uint64)
    cols = k ^ np.uint64(x)
    ny = bin(int(x) & int(z)).count("1") & 3
    sgn = 1.0 - 2.0 * _parity(cols & np.uint64(z))
    return _IPOW[ny] * np.vdot(psi, sgn * psi[cols.astype(np.int64)])


def trotter_state(n, hf_bits, plan_arrays, theta_plan_order):
    """prod_g exp(theta_g A_g) |hf>, generators in plan (execution) order;
    A_g = sum_j c_j P_j with the plan's complex coefficients (anti-Hermitian)."""
    off, xs, zs, cs = plan_arrays
    psi = np.zeros(1 << n, dtype=complex)
    psi[int(hf_bits)] = 1.0
    for g in range(len(off) - 1):
        A = None
        for j in range(off[g], off[g + 1]):
            M = complex(cs[j]) * pauli_sparse(n, int(xs[j]), int(zs[j]))
            A = M if A is None else A + M
        if A is not None:
            psi = expm_multiply(float(theta_plan_order[g]) * A.tocsc(), psi)
    return psi


def energy(n, hf_bits, plan_arrays, theta_plan_order, ham_arrays):
    psi = trotter_state(n, hf_bits, plan_arrays, theta_plan_order)
    x, z, c = ham_arrays
    e = 0.0 + 0.0j
    for xt, zt, ct in zip(x, z, c):
        e += complex(ct) * pauli_expect(n, psi, int(xt), int(zt))
    return e, psi
