"""Pin the CPU oracle (oracle/ffo_oracle.c) before trusting it.

The reference has no code or golden vectors for this path, so
the oracle is pinned by: the SPEC's own examples (KATs, SPEC.md line cited per
test), dense numpy/scipy matrices, a Jordan-Wigner-free fermionic evaluator,
the C++ standard's mt19937_64 known answer, and the reference's one golden
number that touches the path (Eq.-1 assembly, test_fmo.cpp:182-185).
"""
import itertools

import numpy as np
import pytest
import scipy.linalg as sl

from dense import fermion_hamiltonian_dense, ladder_dense, pauli_dense, psum_dense


def test_mt19937_64_known_answer(oracle):
    # C++ standard [rand.predef]: 10000th output of default-seeded mt19937_64
    assert oracle.mt64_nth(5489, 10000) == 9981545732273789042


def test_pauli_mul_kats(oracle):
    # SPEC.md:349 X*Y = iZ ; SPEC.md:350 P*P = I
    k, x, z = oracle.pauli_mul(1, 1, 0, 1, 1)
    assert (k, x, z) == (1, 0, 1)
    k, x, z = oracle.pauli_mul(3, 0b101, 0b110, 0b101, 0b110)
    assert (k, x, z) == (0, 0, 0)


def test_pauli_mul_dense_6q(oracle):
    # random 6-qubit pairs vs 64x64 dense product
    rng = np.random.default_rng(11)
    for _ in range(20):
        x1, z1, x2, z2 = (int(v) for v in rng.integers(0, 64, 4))
        k, x3, z3 = oracle.pauli_mul(6, x1, z1, x2, z2)
        lhs = pauli_dense(6, x1, z1) @ pauli_dense(6, x2, z2)
        assert np.allclose(lhs, (1j ** k) * pauli_dense(6, x3, z3), atol=1e-15)


def test_jw_number_operator(oracle):
    # a+_0 a_0 -> (I - Z_0)/2
    x, z, c = oracle.jw_product(2, [(0, True), (0, False)]).terms()
    assert list(zip(x.tolist(), z.tolist())) == [(0, 0), (0, 1)]
    assert np.allclose(c, [0.5, -0.5])


def test_jw_canonical_anticommutation(oracle):
    # {a+_p, a_q} = delta_pq I for p, q <= 4
    n = 5
    for p, q in itertools.product(range(n), repeat=2):
        s1 = oracle.jw_product(n, [(p, True), (q, False)])
        s2 = oracle.jw_product(n, [(q, False), (p, True)])
        M = psum_dense(n, *s1.terms()) + psum_dense(n, *s2.terms())
        assert np.allclose(M, np.eye(1 << n) * (p == q), atol=1e-14)


def test_jw_matches_fermionic_dense(oracle):
    # JW image of the spin-orbital Hamiltonian == second-quantised matrix
    for m, seed in ((2, 3), (3, 7)):
        h, g = oracle.synthetic_integrals(m, seed)
        H = oracle.hamiltonian_jw(h, g, 0.25)
        assert np.abs(psum_dense(2 * m, *H.terms()) - fermion_hamiltonian_dense(h, g, 0.25)).max() < 1e-13


def test_h2_like_hamiltonian_has_15_terms(oracle):
    # H2/STO-3G JW image has 15 terms. Any 2-orbital Hamiltonian
    # with H2's gerade/ungerade symmetry (h_01 = 0, (00|01) = (11|01) = 0)
    # has that structure; the values below are arbitrary, not H2's.
    h = np.array([[-1.1, 0.0], [0.0, -0.4]])
    g = np.zeros((2, 2, 2, 2))
    vals = {(0, 0, 0, 0): 0.61, (1, 1, 1, 1): 0.63, (0, 0, 1, 1): 0.58, (0, 1, 0, 1): 0.17}
    for (p, q, r, s), v in vals.items():
        for a, b, c, d in ((p, q, r, s), (q, p, r, s), (p, q, s, r), (q, p, s, r),
                           (r, s, p, q), (s, r, p, q), (r, s, q, p), (s, r, q, p)):
            g[a, b, c, d] = v
    H = oracle.hamiltonian_jw(h, g, 0.7)
    assert len(H) == 15
    E_dense = np.linalg.eigvalsh(fermion_hamiltonian_dense(h, g, 0.7))
    assert np.allclose(np.linalg.eigvalsh(psum_dense(4, *H.terms())), E_dense, atol=1e-12)


def test_hf_state(oracle):
    # SPEC.md:407-409
    psi = oracle.hf_state(4, 0b0011)
    assert psi[3] == 1.0 and np.isclose(np.linalg.norm(psi), 1.0)


def test_rotation_kats(oracle):
    rng = np.random.default_rng(5)
    n = 6
    psi = rng.normal(size=64) + 1j * rng.normal(size=64)
    psi /= np.linalg.norm(psi)
    for x, z in ((0b101101, 0b011001), (0, 0b110), (0b1, 0b1), (0b100000, 0)):
        # SPEC.md:416 theta = 0 is the identity
        assert np.array_equal(oracle.apply_pauli_rotation(n, psi, x, z, 0.0), psi)
        # SPEC.md:417 e^{i pi P} = -I
        assert np.allclose(oracle.apply_pauli_rotation(n, psi, x, z, np.pi), -psi, atol=1e-15)
        # SPEC.md:418 vs dense expm
        th = 0.37
        ref = sl.expm(1j * th * pauli_dense(n, x, z)) @ psi
        assert np.abs(oracle.apply_pauli_rotation(n, psi, x, z, th) - ref).max() < 1e-12


def test_expectation_kats(oracle):
    # SPEC.md:425 H = I -> 1 ; SPEC.md:426 Z_0 on |0> -> +1
    I = oracle.PauliSum.from_terms(3, [0], [0], [1.0])
    assert np.isclose(oracle.expectation(3, oracle.hf_state(3, 0b101), I), 1.0)
    Z0 = oracle.PauliSum.from_terms(3, [0], [1], [1.0])
    assert np.isclose(oracle.expectation(3, oracle.hf_state(3, 0), Z0), 1.0)
    # SPEC.md:427 random 5-qubit H, random state vs dense
    rng = np.random.default_rng(9)
    x = rng.integers(0, 32, 40).astype(np.uint64)
    z = rng.integers(0, 32, 40).astype(np.uint64)
    c = rng.normal(size=40)
    H = oracle.PauliSum.from_terms(5, x, z, c)
    psi = rng.normal(size=32) + 1j * rng.normal(size=32)
    psi /= np.linalg.norm(psi)
    ref = np.vdot(psi, psum_dense(5, *H.terms()) @ psi)
    assert abs(oracle.expectation(5, psi, H) - ref) < 1e-12


def test_generators_kats(oracle):
    # H2 (2 e in 4 spin orbitals) -> 3 generators ; :498 no virtuals -> empty
    kind, idx = oracle.build_generators(4, 2)
    assert len(kind) == 3 and sorted(kind.tolist()) == [1, 1, 2]
    kind, _ = oracle.build_generators(4, 4)
    assert len(kind) == 0
    # BASELINE configs
    for n_so, ne, want in ((8, 4, 26), (12, 6, 117), (18, 10, 560)):
        assert len(oracle.build_generators(n_so, ne)[0]) == want


def test_generator_image_is_jw_of_tau_minus_dagger(oracle):
    n = 6
    a = [ladder_dense(n, p, False) for p in range(n)]
    ad = [ladder_dense(n, p, True) for p in range(n)]
    kind, idx = oracle.build_generators(n, 3)
    for k, (i, j, A, B) in zip(kind, idx):
        tau = ad[A] @ a[i] if k == 1 else ad[A] @ ad[B] @ a[j] @ a[i]
        x, z, c = oracle.generator_image(n, k, (i, j, A, B)).terms()
        assert np.allclose(c.real, 0)
        assert np.abs(psum_dense(n, x, z, c) - (tau - tau.T)).max() < 1e-15
        assert len(set(x.tolist())) == 1  # one flip mask per generator


def test_magnitude_order_kats(oracle):
    # SPEC.md:505-507
    assert oracle.magnitude_order([0.1, -0.3]).tolist() == [1, 0]
    assert oracle.magnitude_order([0.0, 0.0, 0.0]).tolist() == [0, 1, 2]
    assert oracle.magnitude_order([0.2, -0.2, 0.5]).tolist() == [2, 0, 1]


@pytest.mark.parametrize("m,ne", [(2, 2), (3, 2), (4, 4)])
def test_energy_trotter_vs_dense_and_fermionic(oracle, m, ne):
    n = 2 * m
    h, g = oracle.synthetic_integrals(m, 100 + m)
    H = oracle.hamiltonian_jw(h, g)
    kind, idx = oracle.build_generators(n, ne)
    amps = np.random.default_rng(m).uniform(-0.4, 0.4, len(kind))
    plan = oracle.magnitude_order(amps)
    e, im, psi = oracle.energy_trotter(n, ne, kind, idx, plan, amps, H, want_state=True)
    ef, psif = oracle.energy_fermionic(h, g, ne, kind, idx, plan, amps, want_state=True)
    a = [ladder_dense(n, p, False) for p in range(n)]
    ad = [ladder_dense(n, p, True) for p in range(n)]
    v = np.zeros(1 << n, complex)
    v[(1 << ne) - 1] = 1
    for gid in plan:
        i, j, A, B = idx[gid]
        tau = ad[A] @ a[i] if kind[gid] == 1 else ad[A] @ ad[B] @ a[j] @ a[i]
        v = sl.expm(amps[gid] * (tau - tau.T)) @ v
    Hd = fermion_hamiltonian_dense(h, g)
    ed = np.vdot(v, Hd @ v).real
    assert abs(e - ed) < 1e-12 and abs(ef - ed) < 1e-12 and abs(im) < 1e-12
    assert np.abs(psi - v).max() < 1e-12 and np.abs(psif - v).max() < 1e-12
    # SPEC.md:448 norm preserved ; SPEC.md:553 variational bound
    assert abs(np.linalg.norm(psi) - 1) < 1e-12
    assert e >= np.linalg.eigvalsh(Hd)[0] - 1e-10


def test_energy_trotter_zero_amplitudes_is_hf_energy(oracle):
    # SPEC.md:514
    m, ne = 4, 4
    h, g = oracle.synthetic_integrals(m, 1)
    H = oracle.hamiltonian_jw(h, g)
    kind, idx = oracle.build_generators(2 * m, ne)
    e, _ = oracle.energy_trotter(2 * m, ne, kind, idx, np.arange(len(kind), dtype=np.int32),
                                 np.zeros(len(kind)), H)
    hf = oracle.hf_state(2 * m, (1 << ne) - 1)
    assert abs(e - oracle.expectation(2 * m, hf, H).real) < 1e-14


def test_fmo_assembly_golden(oracle):
    # reference proj/tests/test_fmo.cpp:182-185 (paper UCCSD:CB column)
    e = oracle.fmo_assemble(3, [-0.026884, -0.026164, -0.026899], [-0.049880, -0.051554, -0.051952])
    assert abs(e - (-0.073439)) <= 1e-9
