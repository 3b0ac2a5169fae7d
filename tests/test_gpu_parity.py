"""GPU parity: the sm_100a path, called through the C-ABI (capi = ctypes over
libfragfield_cuda.so), against the CPU oracle on the same seeded inputs.

Tolerances (north_star): energies <= 1e-10 Hartree absolute, amplitudes
<= 1e-12 max-abs. Full-size configs are checked through size-independent
properties (norm, HF limit, determinism, inverse rotations)."""
import os
import time

import numpy as np
import pytest

import paper_2402_17993_b200 as ff
from paper_2402_17993_b200 import capi, problems

pytestmark = pytest.mark.gpu

E_TOL = 1e-10
A_TOL = 1e-12


@pytest.fixture(scope="module")
def ctx():
    return capi.Context(0)


def oracle_H(oracle, P):
    x, z, c = P.ham_arrays()
    return oracle.PauliSum.from_terms(P.n_qubits, x, z, c)


def upload(ctx, P):
    return (capi.Plan(ctx, P.n_qubits, *P.plan_arrays()), capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays()))


def oracle_energy(oracle, P, theta_canonical, want_state=False):
    kind, idx = oracle.build_generators(P.n_qubits, P.n_elec)
    return oracle.energy_trotter(P.n_qubits, P.n_elec, kind, idx, np.array(P.plan.order, np.int32),
                                 theta_canonical, oracle_H(oracle, P), want_state=want_state)


@pytest.mark.parametrize("n", [2, 3, 6, 11])
def test_pauli_rotation_all_modes_vs_oracle(ctx, oracle, n):
    rng = np.random.default_rng(n)
    dim = 1 << n
    psi = rng.normal(size=(2, dim)) + 1j * rng.normal(size=(2, dim))
    psi /= np.linalg.norm(psi, axis=1, keepdims=True)
    st = capi.State(ctx, n, 2)
    st.upload(psi)
    ref = psi.copy()
    strings = [(0, 1), (1, 0), (1, 3), (dim - 1, dim - 1), (2 % dim, 1), (dim - 2, 5 % dim), (3, 0)]
    for k, (x, z) in enumerate(strings):
        th = 0.3 + 0.17 * k
        st.rotate(x, z, th)
        for b in range(2):
            ref[b] = oracle.apply_pauli_rotation(n, ref[b], x, z, th)
    assert np.abs(st.download() - ref).max() <= A_TOL


@pytest.mark.parametrize("config", [1, 2])
def test_plan_amplitudes_and_energy_vs_oracle(ctx, oracle, config):
    P = problems.config_problem(config)
    plan, ham = upload(ctx, P)
    e_ref, im_ref, psi_ref = oracle_energy(oracle, P, P.thetas[0], want_state=True)
    st = capi.State(ctx, P.n_qubits, 1)
    st.set_basis(P.hf)
    st.apply_plan(plan, P.plan_thetas())
    assert np.abs(st.download()[0] - psi_ref).max() <= A_TOL
    assert abs(st.expectation(ham)[0].real - e_ref) <= E_TOL
    assert abs(capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())[0] - e_ref) <= E_TOL


def test_config2_batch_of_64_vs_oracle(ctx, oracle):
    P = problems.config_problem(2, batch=64)
    plan, ham = upload(ctx, P)
    e = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())
    for b in (0, 17, 63):
        assert abs(e[b] - oracle_energy(oracle, P, P.thetas[b])[0]) <= E_TOL


def test_parameter_shift_set_vs_oracle(ctx, oracle):
    P = problems.config_problem(1)
    plan, ham = upload(ctx, P)
    rows = np.array(ff.parameter_shift_set(list(P.thetas[0]))).reshape(-1, P.n_gen)
    e = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas(rows))
    for r in (0, 1, 2, len(rows) - 1):
        assert abs(e[r] - oracle_energy(oracle, P, rows[r])[0]) <= E_TOL


def test_global_path_matches_smem_path_and_oracle(oracle, monkeypatch):
    # the same 12-qubit problem through the graph-of-kernels path
    monkeypatch.setenv("FFQ_SECTOR", "0")
    monkeypatch.setenv("FFQ_SMEM_MAX_QUBITS", "0")
    gctx = capi.Context(0)
    P = problems.config_problem(2, batch=5)
    plan, ham = upload(gctx, P)
    e_glob = capi.energy_batch(gctx, plan, ham, P.hf, P.plan_thetas())
    monkeypatch.delenv("FFQ_SMEM_MAX_QUBITS")
    sctx = capi.Context(0)
    plan2, ham2 = upload(sctx, P)
    e_smem = capi.energy_batch(sctx, plan2, ham2, P.hf, P.plan_thetas())
    assert np.abs(e_glob - e_smem).max() <= 1e-12
    assert abs(e_glob[3] - oracle_energy(oracle, P, P.thetas[3])[0]) <= E_TOL


def test_18_qubit_energy_vs_oracle(ctx, oracle):
    P = problems.config_problem(3)
    plan, ham = upload(ctx, P)
    t = time.time()
    e_ref = oracle_energy(oracle, P, P.thetas[0])[0]
    e = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())
    assert abs(e[0] - e_ref) <= E_TOL, (e[0], e_ref, time.time() - t)


def test_determinism_across_batch_splits(ctx):
    P = problems.config_problem(3, batch=20)
    plan, ham = upload(ctx, P)
    th = P.plan_thetas()
    full = capi.energy_batch(ctx, plan, ham, P.hf, th)
    parts = np.concatenate([capi.energy_batch(ctx, plan, ham, P.hf, th[i:i + 7]) for i in range(0, 20, 7)])
    single = capi.energy_batch(ctx, plan, ham, P.hf, th[11:12])
    assert np.array_equal(full, parts) and full[11] == single[0]


def test_split_evaluations_bit_identical(ctx):
    # batches below the SM count run each 18-qubit evaluation on up to 16 CTAs
    # (warp sums + block_sum's second-stage tree): the energies must be the
    # one-CTA kernel's, bit for bit, whatever the split
    P = problems.config_problem(3, batch=150)
    plan, ham = upload(ctx, P)
    th = P.plan_thetas()
    full = capi.energy_batch(ctx, plan, ham, P.hf, th)  # 150 rows: one CTA each
    for b in (1, 2, 5, 18, 37, 74):  # splits 16, 16, 16, 8, 4, 2
        part = capi.energy_batch(ctx, plan, ham, P.hf, th[:b])
        assert np.array_equal(part, full[:b]), b


def test_split_launches_back_to_back_random_batches(ctx):
    # role-warp launches keep one arrival ticket per row on the context (the
    # evaluation's last CTA adds the warp sums and clears it) and warm L2 on the
    # idle SMs: forty calls of random sizes back to back, growing and shrinking
    # the ticket buffer's use, each equal to the one-CTA energies bit for bit
    P = problems.config_problem(3, batch=150)
    plan, ham = upload(ctx, P)
    th = P.plan_thetas()
    full = capi.energy_batch(ctx, plan, ham, P.hf, th)
    rng = np.random.default_rng(7)
    for b in rng.integers(1, 148, size=40):
        o = int(rng.integers(0, 150 - b + 1))
        part = capi.energy_batch(ctx, plan, ham, P.hf, th[o:o + b])
        assert np.array_equal(part, full[o:o + b]), (int(b), o)


def test_full_size_properties_18q(ctx):
    P = problems.config_problem(3)
    plan, ham = upload(ctx, P)
    # zero amplitudes -> HF energy = diagonal element
    e0 = capi.energy_batch(ctx, plan, ham, P.hf, np.zeros((1, P.n_gen)))[0]
    st = capi.State(ctx, 18, 1)
    st.set_basis(P.hf)
    assert abs(st.expectation(ham)[0].real - e0) <= 1e-12
    # norm preservation after the full plan
    st.apply_plan(plan, P.plan_thetas())
    psi = st.download()[0]
    assert abs(np.linalg.norm(psi) - 1.0) <= 1e-12
    # particle number and S_z are conserved: support only on 5 alpha + 5 beta
    idx = np.nonzero(np.abs(psi) > 1e-14)[0]
    alpha = np.array([bin(k & 0x15555).count("1") for k in idx])
    beta = np.array([bin(k & 0x2AAAA).count("1") for k in idx])
    assert np.all(alpha == 5) and np.all(beta == 5)


def test_large_state_rotation_roundtrip(ctx):
    # 26 qubits (1 GiB): e^{-i t P} e^{i t P} = I on a random state
    n = 26
    st = capi.State(ctx, n, 1)
    rng = np.random.default_rng(0)
    psi = (rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)) / np.sqrt(2 << n)
    st.upload(psi)
    for x, z in ((0b1010 << 20, 0b11), (1 | (1 << 25), 1 << 3), (0, (1 << 26) - 1), (1, 2)):
        st.rotate(x, z, 0.41)
        st.rotate(x, z, -0.41)
    assert np.abs(st.download()[0] - psi).max() <= A_TOL


def test_error_paths(ctx):
    with pytest.raises(ff.ContractViolation):
        capi.Hamiltonian(ctx, 2, [1], [0], [0.5j])  # non-Hermitian
    with pytest.raises(ff.ContractViolation):
        capi.Plan(ctx, 2, [0, 1], [1], [0], [0.5])  # generator not anti-Hermitian
    P1 = problems.config_problem(1)
    P2 = problems.config_problem(2)
    plan = capi.Plan(ctx, P1.n_qubits, *P1.plan_arrays())
    ham = capi.Hamiltonian(ctx, P2.n_qubits, *P2.ham_arrays())
    with pytest.raises(ff.ContractViolation):
        capi.energy_batch(ctx, plan, ham, P1.hf, P1.plan_thetas())
    with pytest.raises(ff.ContractViolation):
        capi.State(ctx, 1, 1)


def test_cpp_facade_energy_and_vqe(oracle):
    dev = ff.Device(0)
    P = problems.config_problem(1)
    H = ff.DeviceHamiltonian(dev, P.H)
    plan = ff.DevicePlan(dev, P.plan)
    assert plan.n_fused == P.n_gen
    e = ff.energy_trotter(dev, list(P.thetas[0]), plan, H, P.hf)
    assert abs(e - oracle_energy(oracle, P, P.thetas[0])[0]) <= E_TOL
    # config 1: full VQE to convergence (Powell, ftol 1e-8); variational bound
    f = lambda t: ff.energy_trotter(dev, list(t), plan, H, P.hf)  # noqa: E731
    r = ff.vqe_minimize(f, list(P.thetas[0]), "powell")
    assert r.converged and r.energy < e
    from dense import psum_dense

    E0 = np.linalg.eigvalsh(psum_dense(8, *P.H.arrays()))[0]
    assert r.energy >= E0 - 1e-10
    assert dev.kernel_launches() > 0


@pytest.mark.parametrize("config", [2, 3])
def test_execution_paths_agree(monkeypatch, config):
    # dense graph path, support-tracked graph path, persistent per-state path
    P = problems.config_problem(config, batch=6)
    out = {}
    for name, env in (("dense", {"FFQ_SUPPORT": "0", "FFQ_PERSIST": "0", "FFQ_SECTOR": "0"}),
                      ("graph", {"FFQ_SUPPORT": "1", "FFQ_PERSIST": "0", "FFQ_SECTOR": "0"}),
                      ("persistent", {"FFQ_SUPPORT": "1", "FFQ_PERSIST": "1", "FFQ_SECTOR": "0"}),
                      ("sector", {"FFQ_SUPPORT": "1", "FFQ_PERSIST": "0", "FFQ_SECTOR": "1"})):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        monkeypatch.setenv("FFQ_SMEM_MAX_QUBITS", "0")
        c = capi.Context(0)
        plan, ham = upload(c, P)
        out[name] = capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas())
        out[name + "2"] = capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas()[::-1])[::-1]
    for name in ("graph", "persistent", "sector"):
        assert np.abs(out[name] - out["dense"]).max() <= 1e-12
        assert np.array_equal(out[name], out[name + "2"])  # the slab is left clean


def test_dense_random_state_plan_and_expectation_vs_oracle(ctx, oracle):
    # an arbitrary dense state: the support bitmap is rebuilt from the data
    P = problems.make_problem(7, 6, problems.ham_seed(9), batch=1, name="m7e6")
    n = P.n_qubits
    rng = np.random.default_rng(4)
    psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    psi /= np.linalg.norm(psi)
    plan, ham = upload(ctx, P)
    st = capi.State(ctx, n, 1)
    st.upload(psi)
    st.apply_plan(plan, P.plan_thetas())
    ref = psi.copy()
    for gid in P.plan.order:
        x, z, c = P.gens[gid].image.arrays()
        for xx, zz, cc in zip(x, z, c):
            ref = oracle.apply_pauli_rotation(n, ref, int(xx), int(zz), P.thetas[0][gid] * cc.imag)
    assert np.abs(st.download()[0] - ref).max() <= A_TOL
    e = st.expectation(ham)[0].real
    assert abs(e - oracle.expectation(n, ref, oracle_H(oracle, P)).real) <= E_TOL
    # a dense rotation then a support-tracked expectation on the same state
    st.rotate(0b101 << 3, 0b11, 0.3)
    ref = oracle.apply_pauli_rotation(n, ref, 0b101 << 3, 0b11, 0.3)
    assert abs(st.expectation(ham)[0].real - oracle.expectation(n, ref, oracle_H(oracle, P)).real) <= E_TOL


def test_sector_path_18q_vs_oracle_and_dense(monkeypatch, oracle):
    P = problems.config_problem(3, batch=3)
    monkeypatch.setenv("FFQ_SECTOR", "1")
    c = capi.Context(0)
    plan, ham = upload(c, P)
    e = capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas())
    assert abs(e[1] - oracle_energy(oracle, P, P.thetas[1])[0]) <= E_TOL
    monkeypatch.setenv("FFQ_SECTOR", "0")
    c2 = capi.Context(0)
    plan2, ham2 = upload(c2, P)
    assert np.abs(e - capi.energy_batch(c2, plan2, ham2, P.hf, P.plan_thetas())).max() <= 1e-12


def test_cuda_path_matches_golden_fixtures(ctx):
    # tests/golden/energies.json (tools/make_golden.py): energies <= 1e-10,
    # the config-1 state <= 1e-12, through the default execution paths
    import json

    with open(os.path.join(os.path.dirname(__file__), "golden", "energies.json")) as f:
        golden = json.load(f)["configs"]
    for cfg, g in golden.items():
        P = problems.config_problem(int(cfg), batch=len(g["rows"]))
        plan, ham = upload(ctx, P)
        e = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())
        ref = np.array([float.fromhex(r["energy"]) for r in g["rows"]])
        assert np.abs(e - ref).max() <= E_TOL, cfg
        for b, row in enumerate(g["rows"]):
            if "state_re" not in row:
                continue
            st = capi.State(ctx, P.n_qubits, 1)
            st.set_basis(P.hf)
            st.apply_plan(plan, P.plan_thetas()[b:b + 1])
            want = np.array([float.fromhex(v) for v in row["state_re"]]) + 1j * np.array(
                [float.fromhex(v) for v in row["state_im"]])
            assert np.abs(st.download()[0] - want).max() <= A_TOL


@pytest.mark.parametrize("config,rows", [(1, 4), (2, 4), (3, 2)])
def test_scbkt_energies_match_jw(ctx, oracle, config, rows):
    """SPEC.md:361-370 two-qubit reduction on the device: the reduced plan
    (n - 2 qubits; its generators run as per-string rotation passes) gives the
    JW energies of the same theta rows (the Trotter energy is mapping
    independent), and at config 1 the oracle's."""
    J = problems.config_problem(config, batch=rows)
    R = problems.config_problem(config, batch=rows, mapping="scbkt")
    assert R.n_qubits == J.n_qubits - 2
    ej = capi.energy_batch(ctx, *upload(ctx, J), J.hf, J.plan_thetas())
    er = capi.energy_batch(ctx, *upload(ctx, R), R.hf, R.plan_thetas())
    assert np.abs(ej - er).max() <= E_TOL
    if config == 1:
        for b in range(rows):
            ref, _ = oracle_energy(oracle, J, J.thetas[b])
            assert abs(er[b] - ref) <= E_TOL


# ---- parity holes closed in round 2 (VERDICT r01 "Next round" #2) ----------------

def test_config2_all_base_rows_and_256_shift_rows_vs_oracle(ctx, oracle):
    """BASELINE config 2: every one of the 64 seeded theta rows, plus 256
    parameter-shift rows (+-pi/2 on singles and doubles, spread over all
    generators and base rows) from the 15 040-row batched call, against the
    oracle row by row."""
    P = problems.config_problem(2, batch=64)
    plan, ham = upload(ctx, P)
    rows = np.concatenate([np.array(ff.parameter_shift_set(list(t))).reshape(-1, P.n_gen) for t in P.thetas])
    assert rows.shape == (64 * (1 + 2 * 117), 117)
    e = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas(rows))
    per = 1 + 2 * P.n_gen
    base = [b * per for b in range(64)]
    rng = np.random.default_rng(2)
    shift = sorted(set((rng.integers(0, 64, 400) * per + 1 + rng.integers(0, 2 * P.n_gen, 400)).tolist()))[:256]
    assert len(shift) == 256
    H = oracle_H(oracle, P)
    kind, idx = oracle.build_generators(P.n_qubits, P.n_elec)
    order = np.array(P.plan.order, np.int32)
    worst = 0.0
    for r in base + shift:
        ref = oracle.energy_trotter(P.n_qubits, P.n_elec, kind, idx, order, rows[r], H)[0]
        worst = max(worst, abs(e[r] - ref))
    assert worst <= E_TOL, worst


def test_config3_shift_rows_vs_oracle(ctx, oracle):
    """BASELINE config 3 (18 qubits, the headline step): 16 rows of the
    1121-row parameter-shift set -- +-pi/2 on singles (generators 0..39) and on
    doubles, early and late in the magnitude order -- evaluated in the full
    batched call (the benchmark's program: real-amplitude sector evaluator with
    alpha-beta cliques and split-free waves) against the oracle."""
    P = problems.config_problem(3)
    plan, ham = upload(ctx, P)
    rows = np.array(ff.parameter_shift_set(list(P.thetas[0]))).reshape(-1, P.n_gen)
    e = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas(rows))
    pos = np.argsort(P.plan.order)  # plan position of each generator
    gens = [0, 7, 19, 39, 40, 41, 100, 250, 401, 559, int(np.argmin(pos)), int(np.argmax(pos))]
    pick = []
    for g in gens:
        pick += [1 + 2 * g, 2 + 2 * g]
    pick = sorted(set(pick))[:16]
    assert len(pick) == 16
    H = oracle_H(oracle, P)
    kind, idx = oracle.build_generators(P.n_qubits, P.n_elec)
    order = np.array(P.plan.order, np.int32)
    for r in pick:
        ref = oracle.energy_trotter(P.n_qubits, P.n_elec, kind, idx, order, rows[r], H)[0]
        assert abs(e[r] - ref) <= E_TOL, (r, e[r], ref)


def test_sector_state_18q_amplitudes_vs_oracle(ctx, oracle, tmp_path):
    """Amplitude parity of the 18-qubit sector program (ffq_sector_state: the
    product-layout slots after the plan, scattered to natural order) against the
    oracle's state, <= 1e-12 max-abs, for the base row and a +pi/2 shift row;
    and the SPEC.md:459 state dump (LE int64 n + 2^n LE complex doubles) of the
    device state round-trips through write/read_state_dump bit for bit."""
    P = problems.config_problem(3)
    plan, ham = upload(ctx, P)
    rows = np.array(ff.parameter_shift_set(list(P.thetas[0]))).reshape(-1, P.n_gen)[[0, 1]]
    for r in range(2):
        psi, e = capi.sector_state(ctx, plan, ham, P.hf, P.plan_thetas(rows[r:r + 1]), P.n_qubits)
        e_ref, _, psi_ref = oracle_energy(oracle, P, rows[r], want_state=True)
        assert np.abs(psi - psi_ref).max() <= A_TOL
        assert abs(e - e_ref) <= E_TOL
        assert abs(np.linalg.norm(psi) - 1.0) <= 1e-12
    path = str(tmp_path / "psi18.bin")
    ff.write_state_dump(path, P.n_qubits, list(psi))
    raw = open(path, "rb").read()
    assert len(raw) == 8 + 16 * (1 << 18) and int.from_bytes(raw[:8], "little") == 18
    back = np.frombuffer(raw[8:], dtype="<f8").view(np.complex128)
    assert np.array_equal(back, psi)


def test_config5_recipe_20q_compact_vs_oracle(oracle, monkeypatch):
    """BASELINE config 5's recipe (all singles + the first doubles in canonical
    order, random {I,X,Y,Z} Hamiltonian) at 20 qubits / 10 electrons through the
    compact real [alpha][beta] sector layout (the path config 5 takes at 32
    qubits) and through the default path, against the oracle's per-string
    rotations and term-by-term expectation."""
    P = problems.config5_problem(n_doubles=200, n_terms=400, n_qubits=20, n_elec=10)
    off, x, z, c = P.plan_arrays()
    gens = [(x[off[g]:off[g + 1]], z[off[g]:off[g + 1]], c[off[g]:off[g + 1]]) for g in range(len(off) - 1)]
    th = P.plan_thetas()[0]
    oracle.set_threads(os.cpu_count() or 1)
    psi = oracle.hf_state(P.n_qubits, P.hf)
    for (gx, gz, gc), t in zip(gens, th):
        for i in np.lexsort((gz, gx)):  # canonical (x, z) order within a generator
            psi = oracle.apply_pauli_rotation(P.n_qubits, psi, int(gx[i]), int(gz[i]), t * gc[i].imag)
    ref = oracle.expectation(P.n_qubits, psi, oracle_H(oracle, P)).real
    for env in ({"FFQ_COMPACT_MIN": "20"}, {}):
        for k in ("FFQ_COMPACT", "FFQ_COMPACT_MIN", "FFQ_SECTOR"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        c2 = capi.Context(0)
        plan, ham = upload(c2, P)
        e = capi.energy_batch(c2, plan, ham, P.hf, P.plan_thetas())[0]
        assert abs(e - ref) <= E_TOL, (env, e, ref)
        del plan, ham, c2
