"""Dense-matrix reference helpers (numpy/scipy) used to pin the oracle at
<= 10 qubits. Test infrastructure only. Conventions: qubit 0 = least
significant bit of the basis index."""
import numpy as np

I2 = np.eye(2, dtype=complex)
X = np.array([[0, 1], [1, 0]], dtype=complex)
Y = np.array([[0, -1j], [1j, 0]], dtype=complex)
Z = np.array([[1, 0], [0, -1]], dtype=complex)


def pauli_dense(n, x, z):
    """Dense matrix of the phase-free string (x, z); Y where both bits set."""
    m = np.array([[1.0 + 0j]])
    for q in range(n - 1, -1, -1):  # kron: most significant qubit first
        xb, zb = (int(x) >> q) & 1, (int(z) >> q) & 1
        s = Y if (xb and zb) else X if xb else Z if zb else I2
        m = np.kron(m, s)
    return m


def psum_dense(n, xs, zs, cs):
    M = np.zeros((1 << n, 1 << n), dtype=complex)
    for x, z, c in zip(xs, zs, cs):
        M += c * pauli_dense(n, x, z)
    return M


def ladder_dense(n, p, dagger):
    """Fermionic a_p / a+_p on determinants, built from occupation bits with
    the Z_{<p} parity (independent of any Pauli algebra)."""
    dim = 1 << n
    M = np.zeros((dim, dim))
    for k in range(dim):
        occ = (k >> p) & 1
        if dagger and occ == 0 or (not dagger) and occ == 1:
            sign = (-1) ** bin(k & ((1 << p) - 1)).count("1")
            M[k ^ (1 << p), k] = sign
    return M


def fermion_hamiltonian_dense(h, g, e_const=0.0):
    m = h.shape[0]
    n = 2 * m
    a = [ladder_dense(n, p, False) for p in range(n)]
    ad = [ladder_dense(n, p, True) for p in range(n)]
    H = e_const * np.eye(1 << n)
    for p in range(n):
        for q in range(n):
            if p % 2 == q % 2:
                H = H + h[p // 2, q // 2] * ad[p] @ a[q]
    for p in range(n):
        for q in range(n):
            for r in range(n):
                for s in range(n):
                    if p % 2 != r % 2 or q % 2 != s % 2:
                        continue
                    v = g[p // 2, r // 2, q // 2, s // 2]
                    if v != 0.0:
                        H = H + 0.5 * v * ad[p] @ ad[q] @ a[s] @ a[r]
    return H
