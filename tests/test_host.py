"""Host-side logic of the product (C++ operator API via pybind11, no device):
compared term-by-term against the independent C oracle."""
import ctypes
import os

import numpy as np
import pytest

import paper_2402_17993_b200 as ff
from paper_2402_17993_b200 import capi, problems


@pytest.mark.parametrize("m,ne", [(2, 2), (4, 4), (6, 6), (9, 10)])
def test_hamiltonian_and_generators_match_oracle(oracle, m, ne):
    seed = problems.ham_seed(1) + m
    h, g = ff.synthetic_integrals(m, seed)
    ho, go = oracle.synthetic_integrals(m, seed)
    assert np.array_equal(h, ho) and np.array_equal(g, go)  # bitwise: same pinned RNG mapping
    x, z, c = ff.qubit_hamiltonian(h, g, ne).arrays()
    xo, zo, co = oracle.hamiltonian_jw(ho, go).terms()
    assert np.array_equal(x, xo) and np.array_equal(z, zo)
    assert np.abs(c - co).max() < 1e-13
    gens = ff.build_generators(2 * m, ne)
    kind, idx = oracle.build_generators(2 * m, ne)
    assert len(gens) == len(kind)
    for gen in gens[:: max(1, len(gens) // 40)]:
        e = gen.exc
        assert (e.kind, e.i, e.j, e.a, e.b) == (kind[gen.id], *idx[gen.id])
        gx, gz, gc = gen.image.arrays()
        ox, oz, oc = oracle.generator_image(2 * m, kind[gen.id], idx[gen.id]).terms()
        assert np.array_equal(gx, ox) and np.array_equal(gz, oz) and np.abs(gc - oc).max() < 1e-15


def test_uniform_vector_matches_oracle(oracle):
    a = np.array(ff.uniform_vector(77, 1000, -0.1, 0.1))
    assert np.array_equal(a, oracle.uniform_array(77, 1000, -0.1, 0.1))
    assert a.min() >= -0.1 and a.max() < 0.1


def test_magnitude_order_matches_oracle(oracle):
    P = problems.config_problem(2)
    assert list(P.plan.order) == oracle.magnitude_order(P.thetas[0]).tolist()
    gens = ff.build_generators(4, 2)
    assert list(ff.magnitude_order(gens, [0.1, -0.3, 0.0], 4).order) == [1, 0, 2]


def test_pauli_mul_matches_oracle(oracle):
    rng = np.random.default_rng(3)
    for _ in range(200):
        n = int(rng.integers(1, 20))
        x1, z1, x2, z2 = (int(v) for v in rng.integers(0, 1 << n, 4))
        k, p = ff.pauli_mul(ff.PauliString(n, x1, z1), ff.PauliString(n, x2, z2))
        assert (k, p.x, p.z) == oracle.pauli_mul(n, x1, z1, x2, z2)


def test_jordan_wigner_api():
    s = ff.jordan_wigner([(1.0, [(0, True), (0, False)])], 2)
    assert s.to_text().split("\n")[:2] == ["0.5 0 II", "-0.5 0 ZI"]
    t = ff.PauliSum.from_text(s.to_text())
    assert np.array_equal(t.arrays()[0], s.arrays()[0])
    with pytest.raises(ff.ContractViolation):
        ff.jordan_wigner([(1.0, [(5, True)])], 4)
    assert ff.PauliString.parse("XZIY").letters() == "XZIY"
    assert ff.PauliString.parse("XZIY").x == 0b1001


def test_plan_compile_fuses_every_uccsd_generator():
    for c in (1, 2, 3):
        P = problems.config_problem(c)
        st = capi.plan_compile_stats(P.n_qubits, *P.plan_arrays())
        assert st["fused"] == P.n_gen and st["string_ops"] == 0 and st["pattern_pairs"] == P.n_gen
        n = P.n_qubits
        n_single = sum(1 for gen in P.gens if gen.exc.kind == 1)
        # singles update 1/4 of the pairs' index space (pattern 10 <-> 01), doubles 1/16
        assert st["pair_updates"] == n_single * (1 << (n - 2)) + (P.n_gen - n_single) * (1 << (n - 4))


def test_plan_compile_falls_back_to_strings_for_noncommuting_generator():
    # X0 and Y0 Z1 share no flip mask pattern that commutes -> string mode
    off = np.array([0, 2], np.int64)
    x = np.array([1, 1], np.uint64)
    z = np.array([0, 3], np.uint64)
    st = capi.plan_compile_stats(2, off, x, z, np.array([0.3j, 0.2j]))
    assert st["fused"] == 0 and st["string_ops"] == 2
    with pytest.raises(ff.ContractViolation):
        capi.plan_compile_stats(2, off, x, z, np.array([0.3, 0.2j]))  # not anti-Hermitian


def test_ham_compile_stats_and_hermiticity():
    P = problems.config_problem(3)
    st = capi.ham_compile_stats(18, *P.ham_arrays())
    assert st["groups"] == 1621 and st["terms"] == 9316
    with pytest.raises(ff.ContractViolation):
        capi.ham_compile_stats(2, [1], [0], [0.5j])


def test_capi_library_exports_every_header_symbol():
    L = ctypes.CDLL(ff.native_library_path())
    syms = capi.header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    assert capi.lib().ffq_version() == 1


def test_no_device_fails_loudly():
    if ff.Device.count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(ff.DeviceError):
        ff.Device(0)
    h = ctypes.c_void_p()
    assert capi.lib().ffq_ctx_create(0, ctypes.byref(h)) == capi.FFQ_ENODEV


def test_optimizers_quadratic_and_rosenbrock():
    c = np.array([0.3, -1.2, 2.0])
    f = lambda x: float(np.sum((np.asarray(x) - c) ** 2))  # noqa: E731
    for meth in ("powell", "neldermead"):
        r = ff.vqe_minimize(f, [0.0, 0.0, 0.0], meth)
        assert r.converged and np.abs(np.array(r.x) - c).max() < 1e-3 and r.n_evals < 2000
    rosen = lambda x: (1 - x[0]) ** 2 + 100 * (x[1] - x[0] ** 2) ** 2  # noqa: E731
    o = ff.OptimizerOptions()
    o.ftol = 1e-14
    o.xtol = 1e-9
    r = ff.powell_minimize(rosen, [-1.2, 1.0], o)
    assert np.abs(np.array(r.x) - 1).max() < 1e-5


def test_exact_gradient_rule_on_trig_polynomial():
    # E(t) with frequencies {1, 2}: the four-term rule is exact
    rng = np.random.default_rng(0)
    a = rng.normal(size=(3, 5))

    def E(th):
        th = np.asarray(th)
        return float(sum(a[0, k] * np.cos(th[k]) + a[1, k] * np.sin(th[k]) + a[2, k] * np.sin(2 * th[k] + 0.3)
                         for k in range(5)))

    th = rng.normal(size=5)
    rows = np.array(ff.exact_gradient_set(list(th))).reshape(-1, 5)
    g = ff.exact_gradient_from_energies([E(r) for r in rows], 5)
    ga = [-a[0, k] * np.sin(th[k]) + a[1, k] * np.cos(th[k]) + 2 * a[2, k] * np.cos(2 * th[k] + 0.3) for k in range(5)]
    assert np.abs(np.array(g) - ga).max() < 1e-12
    ps = np.array(ff.parameter_shift_set(list(th))).reshape(-1, 5)
    assert ps.shape == (11, 5) and np.array_equal(ps[0], th)


def test_bfgs_with_batched_objective():
    c = np.array([0.2, -0.1])

    def fb(X, B):
        X = np.asarray(X).reshape(B, 2)
        return list(np.sum(np.sin(X - c) ** 2, axis=1))

    r = ff.bfgs_minimize(fb, [0.5, 0.4])
    assert r.converged and np.abs(np.array(r.x) - c).max() < 1e-4


def test_fmo_assembly_matches_reference_golden():
    # proj/tests/test_fmo.cpp:182-185
    mono = {"1": -0.026884, "2": -0.026164, "3": -0.026899}
    dim = {"21": -0.049880, "31": -0.051554, "32": -0.051952}
    assert abs(ff.assemble_two_body(3, mono, dim) - (-0.073439)) <= 1e-9
    assert ff.dimer_labels(3) == ["21", "31", "32"]
    bad = dict(dim)
    bad.pop("21")
    with pytest.raises(ff.ContractViolation):
        ff.assemble_two_body(3, mono, bad)


@pytest.mark.parametrize("g", [0, 1, 2, 3])
def test_shard_schedule_is_a_valid_swap_sequence(g):
    P = problems.config_problem(3)
    ip, fp, ns, st = capi.shard_schedule(18, g, *P.plan_arrays())
    assert sorted(ip.tolist()) == list(range(18)) and sorted(fp.tolist()) == list(range(18))
    assert st == P.n_gen + ns  # every generator applied once, preceded by its swaps
    # the initial global qubits are the least-flipped logical qubits
    uses = np.zeros(18, int)
    for gen in P.gens:
        x = int(gen.image.arrays()[0][0])
        uses += [(x >> q) & 1 for q in range(18)]
    glob = [q for q in range(18) if ip[q] >= 18 - g]
    assert all(uses[q] <= min(uses[[r for r in range(18) if r not in glob]]) for q in glob)
    # local positions ascend with use (hot qubits sit high: long contiguous runs per generator pass)
    at = {int(ip[q]): q for q in range(18)}
    local_uses = [uses[at[pos]] for pos in range(18 - g)]
    assert local_uses == sorted(local_uses)
    if g == 0:
        assert ns == 0


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_sector_program_emulation_matches_oracle(oracle, cfg):
    """The real one-CTA sector program's expectation tables (product slot
    layout + anchored string blocks at 18 qubits, generic rows below), run on
    the host exactly as k_sector_eval_real reads them, against the oracle's
    term-by-term <psi|H|psi> on a random real sector state."""
    P = problems.config_problem(cfg)
    n = P.n_qubits
    k = np.arange(1 << n, dtype=np.int64)
    am = sum(1 << q for q in range(0, n, 2))
    pop = np.vectorize(lambda v: bin(v).count("1"))
    pa, pb = pop(k & am), pop(k & ~am & ((1 << n) - 1))
    na, nb = bin(P.hf & am).count("1"), bin(P.hf & ~am).count("1")
    rng = np.random.default_rng(cfg)
    psi = np.where((pa == na) & (pb == nb), rng.standard_normal(1 << n), 0.0)
    psi /= np.linalg.norm(psi)
    r = capi.sector_emulate(n, P.plan_arrays(), P.ham_arrays(), P.hf, psi)
    H = oracle.PauliSum.from_terms(n, *P.ham_arrays())
    ref = oracle.expectation(n, psi.astype(np.complex128), H)
    assert abs(r["energy"] - ref.real) <= 1e-12
    assert r["table_violations"] == 0  # steps race-free, every slot in bounds
    assert r["closure_size"] == int(((pa == na) & (pb == nb)).sum())
    if cfg == 3:  # 18 qubits: (5a, 5b) sector = 126 x 126 strings, stride 127
        assert r["product"] == 1 and r["slots"] == 126 * 127
        assert r["block_pairs"] + r["clique_pairs"] >= 0.8 * r["exp_pairs"] and r["units"] > 0
        # the alpha-beta pairs (36 alpha x 36 beta single excitations, 35 x 70 pairs each) all factorise
        assert r["clique_pairs"] == 36 * 36 * 35 * 70
    else:  # small closures keep the natural layout (128-thread program)
        assert r["product"] == 0 and r["block_pairs"] == 0


@pytest.mark.parametrize("n,t,seed", [(16, 12, 0), (16, 12, 1), (20, 12, 5), (16, 5, 2), (16, 3, 3), (16, 2, 4),
                                      (8, 12, 6)])
def test_rotation_groups_cover_and_partition(n, t, seed):
    """Host logic of the fused rotation runs (build_rot_runs behind
    ffq_state_apply_pauli_rotations): a run is a greedy stretch of >= 2
    rotations whose flip masks, with the low 5 qubits, fit in min(n, t) qubits
    (run_q = that union filled with the lowest free qubits); each group's masks
    (in tile coordinates, pext by run_q) lie in the span of a reduced-echelon
    basis of 3 vectors (cx = coordinates), pivots ascending below t, and the
    cosets k ^ span{b} (pivot bits of k clear) partition the tile."""
    rng = np.random.default_rng(seed)
    tt = min(n, t)
    x = np.where(rng.random(60) < 0.6, rng.integers(0, 1 << min(tt, n), size=60),
                 rng.integers(1, 1 << n, size=60)).astype(np.uint64)
    x[10:14] = 0  # diagonal rotations join any group
    x[20:26] = [1 << (n - 1), 1 << (n - 2), (1 << (n - 1)) | 1, 3 << (n - 3), 1 << (n - 1), 2]  # high qubits
    run_of, group_of, cx, run_q, basis, piv = capi.rotation_groups(n, t, x)
    low = (1 << min(5, tt)) - 1
    want = np.full(len(x), -1)
    want_q = np.zeros(len(x), np.uint64)
    i, nrun = 0, 0
    while i < len(x) and tt >= 3:
        U, e = low, i
        while e < len(x) and bin(U | int(x[e])).count("1") <= tt:
            U |= int(x[e])
            e += 1
        if e - i < 2:
            i = max(i + 1, e)
            continue
        q, bit = U, 0
        while bin(q).count("1") < tt:
            q |= 1 << bit
            bit += 1
        want[i:e] = nrun
        want_q[i:e] = q
        nrun += 1
        i = e
    assert np.array_equal(run_of, want)
    assert np.array_equal(run_q, want_q)
    assert np.all((group_of >= 0) == (run_of >= 0))
    assert np.all(np.diff(group_of[group_of >= 0]) >= 0)  # groups are consecutive

    def pext(v, m):
        r, o = 0, 0
        while m:
            lsb = m & -m
            if v & lsb:
                r |= 1 << o
            m ^= lsb
            o += 1
        return r

    for g in range(len(basis)):
        b, p = [int(v) for v in basis[g]], [int(v) for v in piv[g]]
        assert p == sorted(p) and len(set(p)) == 3 and max(p) < tt
        for k in range(3):
            assert (b[k] >> p[k]) & 1
            assert all(not ((b[j] >> p[k]) & 1) for j in range(3) if j != k)
        for r in np.nonzero(group_of == g)[0]:
            span = 0
            for k in range(3):
                if (cx[r] >> k) & 1:
                    span ^= b[k]
            assert span == pext(int(x[r]), int(run_q[r]))
        if tt <= 6:
            seen = np.zeros(1 << tt, int)
            pm = sum(1 << v for v in p)
            for k in range(1 << tt):
                if k & pm:
                    continue
                for c in range(8):
                    off = (b[0] if c & 1 else 0) ^ (b[1] if c & 2 else 0) ^ (b[2] if c & 4 else 0)
                    seen[k ^ off] += 1
            assert np.all(seen == 1)


def test_bfgs_line_search_failure_is_not_convergence():
    """A line search that finds no decrease while the gradient is not small
    (here: the objective lies about its own gradient, so BFGS walks uphill)
    must come back UNconverged (best-so-far flagged
    unconverged), after one steepest-descent restart -- not as converged."""
    def fb(X, B):
        X = np.asarray(X).reshape(B, 2)
        if B == 1:  # energies: a bowl at 0
            return list(np.sum(X ** 2, axis=1))
        # gradient rows (4 per parameter): make the four-term rule return -grad
        return list(-np.sum(np.sin(X) ** 2, axis=1))

    r = ff.bfgs_minimize(fb, [0.5, -0.3])
    assert not r.converged
    assert r.energy <= 0.5 ** 2 + 0.3 ** 2  # best-so-far, never worse than the start


def test_sector_program_emulation_on_a_non_molecular_hamiltonian(oracle):
    """A random half of the config-3 Hamiltonian is not molecular: the clique
    factorisation check can refuse alpha-beta groups, which then stay in the
    anchored blocks or generic rows. The tables compiled for it, run on the host
    as the kernel reads them, must still give the oracle's term-by-term
    <psi|H|psi> on a random real sector state, race-free and in bounds."""
    P = problems.config_problem(3)
    n = P.n_qubits
    x, z, co = P.ham_arrays()
    pick = np.random.default_rng(18).random(len(x)) < 0.5
    k = np.arange(1 << n, dtype=np.uint64)
    am = np.uint64(sum(1 << q for q in range(0, n, 2)))
    pa, pb = np.bitwise_count(k & am), np.bitwise_count(k & ~am)
    na, nb = bin(P.hf & int(am)).count("1"), bin(P.hf & ~int(am)).count("1")
    psi = np.where((pa == na) & (pb == nb), np.random.default_rng(3).standard_normal(1 << n), 0.0)
    psi /= np.linalg.norm(psi)
    r = capi.sector_emulate(n, P.plan_arrays(), (x[pick], z[pick], co[pick]), P.hf, psi)
    ref = oracle.expectation(n, psi.astype(np.complex128), oracle.PauliSum.from_terms(n, x[pick], z[pick], co[pick]))
    assert abs(r["energy"] - ref.real) <= 1e-12
    assert r["table_violations"] == 0 and r["product"] == 1
    assert r["clique_pairs"] + r["block_pairs"] > 0


@pytest.mark.parametrize("case", ["config1", "config2", "config5_14q", "uccsd_10q_open"])
def test_compact_program_emulation_matches_oracle(oracle, case):
    """The compact real sector program (csrc/ffq_compact.inl: row / column lists
    per generator, Pauli-term groups with every pair once), compiled and run on
    the host from the lists the kernels read, against the oracle's Trotter energy
    (per-string rotations, term-by-term expectation): molecular Hamiltonians
    (multi-term groups), the config-5 recipe (one-term groups of random strings,
    odd-Y terms dropped) and an open-shell sector (N_alpha != N_beta)."""
    if case == "config1":
        P = problems.config_problem(1)
    elif case == "config2":
        P = problems.config_problem(2)
    elif case == "config5_14q":
        P = problems.config5_problem(n_doubles=120, n_terms=300, n_qubits=14, n_elec=6)
    else:
        P = problems.make_problem(5, 5, problems.ham_seed(9, 5))
    off, x, z, c = P.plan_arrays()
    th = P.plan_thetas()[0]
    r = capi.compact_emulate(P.n_qubits, (off, x, z, c), P.ham_arrays(), P.hf, th)
    assert r["eligible"] == 1 and r["violations"] == 0
    na, nb = bin(P.hf & 0x55555555).count("1"), bin(P.hf & 0xAAAAAAAA).count("1")
    from math import comb
    assert (r["alpha_strings"], r["beta_strings"]) == (comb(P.n_qubits // 2, na), comb(P.n_qubits // 2, nb))
    psi = oracle.hf_state(P.n_qubits, P.hf)
    for g in range(len(off) - 1):
        gx, gz, gc = x[off[g]:off[g + 1]], z[off[g]:off[g + 1]], c[off[g]:off[g + 1]]
        for i in np.lexsort((gz, gx)):  # canonical (x, z) order within a generator
            psi = oracle.apply_pauli_rotation(P.n_qubits, psi, int(gx[i]), int(gz[i]), th[g] * gc[i].imag)
    hx, hz, hc = P.ham_arrays()
    ref = oracle.expectation(P.n_qubits, psi, oracle.PauliSum.from_terms(P.n_qubits, hx, hz, hc)).real
    assert abs(r["energy"] - ref) <= 1e-11, (r["energy"], ref)
    assert r["generator_pairs"] > 0 and r["term_groups"] > 0


def test_compact_program_eligibility():
    # a generator that does not conserve both spin counts (alpha -> beta single
    # excitation image) and a non-fused plan are refused: eligible = 0, no energy
    P = problems.config_problem(1)
    off, x, z, c = P.plan_arrays()
    bad_off = np.array([0, 2], np.int64)  # X0 X1 / Y0 Y1-like pair: flips one alpha and one beta qubit
    bx = np.array([0b11, 0b11], np.uint64)
    bz = np.array([0b01, 0b10], np.uint64)
    bc = np.array([0.5j, -0.5j])
    r = capi.compact_emulate(P.n_qubits, (bad_off, bx, bz, bc), P.ham_arrays(), P.hf, np.array([0.3]))
    assert r["eligible"] == 0
    r = capi.compact_emulate(P.n_qubits, (off, x, z, c), P.ham_arrays(), P.hf, P.plan_thetas()[0])
    assert r["eligible"] == 1
