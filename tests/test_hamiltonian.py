"""f1: the hamiltonian module's AO -> MO transformation and
frozen-core contraction on CPU, against the SPEC examples:
C = I identity, orthogonal-rotation invariants, a brute-force O(N^8)
transform, n_frozen = 0 identity, the frozen-core CAS-CI identity, and
<HF|H|HF> + E_const consistency."""
import itertools

import numpy as np
import pytest

import paper_2402_17993_b200 as ff


def _ao(n, seed):
    h, g = ff.synthetic_integrals(n, seed)
    return np.asarray(h), np.asarray(g)


def _orthogonal(n, seed):
    q, r = np.linalg.qr(np.random.default_rng(seed).normal(size=(n, n)))
    return q * np.sign(np.diag(r))


def test_identity_coefficients_give_ao_integrals():
    h, g = _ao(5, 11)
    hm, gm, ec = ff.ao_to_mo(h, g, np.eye(5), 0.7)
    assert np.array_equal(hm, h) and np.array_equal(gm, g) and ec == 0.7


def test_orthogonal_rotation_invariants():
    h, g = _ao(6, 12)
    C = _orthogonal(6, 3)
    hm, gm, _ = ff.ao_to_mo(h, g, C)
    assert abs(np.trace(hm) - np.trace(h)) <= 1e-12  # similarity invariance of the trace
    assert abs(np.linalg.norm(gm) - np.linalg.norm(g)) <= 1e-12
    # and back: C^T applied to the MO integrals recovers the AO ones
    h2, g2, _ = ff.ao_to_mo(hm, gm, C.T)
    assert np.abs(h2 - h).max() <= 1e-12 and np.abs(g2 - g).max() <= 1e-12


def test_matches_brute_force_transform_and_folds_embedding():
    n, m = 4, 3
    h, g = _ao(n, 13)
    C = np.random.default_rng(4).normal(size=(n, m))
    V = np.random.default_rng(5).normal(size=(n, n))
    V = V + V.T
    hm, gm, _ = ff.ao_to_mo(h, g, C, 0.0, V)
    ref_h = np.zeros((m, m))
    ref_g = np.zeros((m, m, m, m))
    for p, q in itertools.product(range(m), repeat=2):
        ref_h[p, q] = sum(C[a, p] * (h[a, b] + V[a, b]) * C[b, q] for a in range(n) for b in range(n))
    for p, q, r, s in itertools.product(range(m), repeat=4):  # naive O(N^8)
        v = 0.0
        for a, b, c, d in itertools.product(range(n), repeat=4):
            v += C[a, p] * C[b, q] * C[c, r] * C[d, s] * g[a, b, c, d]
        ref_g[p, q, r, s] = v
    assert np.abs(hm - ref_h).max() <= 1e-12
    assert np.abs(gm - ref_g).max() <= 1e-12


def test_freeze_core_zero_is_identity_and_errors():
    h, g = _ao(4, 14)
    he, ge, ec, ef, ne = ff.freeze_core(h, g, 0.25, 0, 4)
    assert np.array_equal(he, h) and np.array_equal(ge, g) and ef == 0.0 and ec == 0.25 and ne == 4
    with pytest.raises(ff.ContractViolation):
        ff.freeze_core(h, g, 0.0, 3, 4)  # 3 frozen orbitals > 2 occupied
    with pytest.raises(ff.ContractViolation):
        ff.freeze_core(h, g, 0.0, -1, 4)


def _sector_matrix(H, n, states):
    """<i|H|j> on a list of basis states (qubit 0 = LSB), from the Pauli terms."""
    x, z, c = H.arrays()
    pos = {k: i for i, k in enumerate(states)}
    M = np.zeros((len(states), len(states)), complex)
    for xx, zz, cc in zip(x, z, c):
        ny = bin(int(xx) & int(zz)).count("1")
        for j, k in enumerate(states):
            t = k ^ int(xx)
            if t in pos:  # P|k> = i^ny (-1)^popc(k & z) |k ^ x>
                M[pos[t], j] += cc * (1j) ** ny * (-1) ** bin(k & int(zz)).count("1")
    return M


def _states(m, na, nb, fixed=0):
    out = []
    for a in itertools.combinations(range(m), na):
        for b in itertools.combinations(range(m), nb):
            k = sum(1 << (2 * p) for p in a) | sum(1 << (2 * p + 1) for p in b)
            if k & fixed == fixed:
                out.append(k)
    return out


def test_frozen_core_casci_equals_full_space_with_core_occupied():
    """CAS-CI on the frozen-core Hamiltonian + E_frozen equals the
    full-space CAS-CI with the core doubly occupied (12 spin orbitals, one core
    orbital); and <HF|H|HF> + E_const agree between the two."""
    m, ne = 6, 6
    h, g = _ao(m, 15)
    C = _orthogonal(m, 6)
    hm, gm, ec = ff.ao_to_mo(h, g, C, 0.3)
    Hfull = ff.qubit_hamiltonian(hm, gm, ne, ec)
    full_states = _states(m, 3, 3, fixed=0b11)  # orbital 0 doubly occupied
    Mf = _sector_matrix(Hfull, 2 * m, full_states)
    assert np.abs(Mf - Mf.conj().T).max() <= 1e-12
    he, ge, ec2, ef, na = ff.freeze_core(hm, gm, ec, 1, ne)
    assert na == 4
    Hfr = ff.qubit_hamiltonian(he, ge, na, ec2)
    Ma = _sector_matrix(Hfr, 2 * (m - 1), _states(m - 1, 2, 2))
    e_full = np.linalg.eigvalsh(Mf)[0]
    e_froz = np.linalg.eigvalsh(Ma)[0]
    assert abs(e_full - e_froz) <= 1e-9
    # HF determinants: lowest orbitals doubly occupied
    hf_full = full_states.index((1 << ne) - 1)
    hf_act = _states(m - 1, 2, 2).index((1 << na) - 1)
    assert abs(Mf[hf_full, hf_full].real - Ma[hf_act, hf_act].real) <= 1e-12
