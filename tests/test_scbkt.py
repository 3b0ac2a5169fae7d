"""SPEC.md:361-370 reduce_two_qubits (SCBKT two-qubit reduction): dense
spectral checks against the JW image (the SPEC's own property), the H2-sized
example, and mapping independence of the Trotterised UCCSD energy. Host only."""
import numpy as np
import pytest
import scipy.linalg

import paper_2402_17993_b200 as ff
from paper_2402_17993_b200 import problems

from dense import psum_dense


def _dense(ps, n):
    x, z, c = ps.arrays()
    return psum_dense(n, x, z, c)


def _apply(ps, psi):
    """A psi for a Pauli sum A: P|k> = i^|x&z| (-1)^popc(k&z) |k ^ x>."""
    k = np.arange(psi.size)
    out = np.zeros_like(psi)
    x, z, c = ps.arrays()
    for xx, zz, cc in zip(x.tolist(), z.tolist(), c):
        sgn = 1.0 - 2.0 * (np.bitwise_count(k & zz) & 1)
        out[k ^ xx] += cc * (1j ** bin(xx & zz).count("1")) * sgn * psi
    return out


def _parity_sector(n, na, nb):
    am = sum(1 << q for q in range(0, n, 2))
    k = np.arange(1 << n)
    pa = np.array([bin(v & am).count("1") for v in k])
    pt = np.array([bin(v).count("1") for v in k])
    return np.nonzero(((pa - na) % 2 == 0) & ((pt - na - nb) % 2 == 0))[0]


@pytest.mark.parametrize("m,ne", [(2, 2), (3, 2), (4, 4), (5, 6)])
def test_reduced_spectrum_equals_jw_on_parity_sector(m, ne):
    h, g = ff.synthetic_integrals(m, problems.ham_seed(7) + m)
    H = ff.qubit_hamiltonian(h, g, ne)
    na, nb = (ne + 1) // 2, ne // 2
    R = ff.reduce_two_qubits(H, 2 * m, na, nb)
    assert R.is_hermitian(1e-12)
    Hd = _dense(H, 2 * m)
    sec = _parity_sector(2 * m, na, nb)
    ej = np.linalg.eigvalsh(Hd[np.ix_(sec, sec)])
    er = np.linalg.eigvalsh(_dense(R, 2 * m - 2))
    assert len(ej) == len(er) == 1 << (2 * m - 2)
    assert np.abs(ej - er).max() <= 1e-10


def test_h2_sized_example_ground_energy():
    # 4 spin orbitals, 1 alpha 1 beta -> 2-qubit Hamiltonian with
    # the ground energy of the JW image in that sector
    h, g = ff.synthetic_integrals(2, problems.ham_seed(7))
    H = ff.qubit_hamiltonian(h, g, 2)
    R = ff.reduce_two_qubits(H, 4, 1, 1)
    assert R.n_qubits == 2
    k = np.arange(16)
    sec = [v for v in k if bin(v & 0b0101).count("1") == 1 and bin(v & 0b1010).count("1") == 1]
    e_jw = np.linalg.eigvalsh(_dense(H, 4)[np.ix_(sec, sec)])[0]
    assert abs(np.linalg.eigvalsh(_dense(R, 2))[0] - e_jw) <= 1e-12


def test_hf_state_maps_to_reduced_basis_state():
    P = problems.config_problem(2)
    R = problems.config_problem(2, mapping="scbkt")
    e = []
    for Q in (P, R):
        psi = np.zeros(1 << Q.n_qubits, complex)
        psi[Q.hf] = 1.0
        e.append(_apply(Q.H, psi)[Q.hf].real)
    assert abs(e[0] - e[1]) <= 1e-12


def test_non_conserving_operator_is_rejected():
    op = ff.PauliSum(8)
    op.add(ff.PauliString.parse("XIIIIIII"), 1.0)  # flips mode 0: changes both parities
    with pytest.raises(ff.ContractViolation):
        ff.reduce_two_qubits(op, 8, 2, 2)


@pytest.mark.parametrize("cfg", [1, 2])
def test_trotter_energy_is_mapping_independent(cfg):
    # each generator's strings commute, so exp(theta A_g) is exact in any
    # encoding: the SCBKT plan must give the JW energies. A_g^3 = -A_g, so
    # exp(t A) psi = psi + sin t A psi + (1 - cos t) A^2 psi.
    out = []
    for mp in ("jw", "scbkt"):
        P = problems.config_problem(cfg, mapping=mp)
        psi = np.zeros(1 << P.n_qubits, complex)
        psi[P.hf] = 1.0
        th = P.thetas[0]
        imgs = P.images if P.images is not None else [gn.image for gn in P.gens]
        for gid in P.plan.order:
            a1 = _apply(imgs[gid], psi)
            psi = psi + np.sin(th[gid]) * a1 + (1 - np.cos(th[gid])) * _apply(imgs[gid], a1)
        out.append(np.vdot(psi, _apply(P.H, psi)).real)
    assert abs(out[0] - out[1]) <= 1e-12
