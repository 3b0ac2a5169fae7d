"""Edge cases of the C-ABI on the GPU, each checked against the CPU oracle:
empty batches and Hamiltonians, plans without generators, identity-only H,
non-UCCSD generators (string fallback) through every execution path, and the
2-pi periodicity of exp(theta A)."""
import os

import numpy as np
import pytest

from paper_2402_17993_b200 import capi, problems

pytestmark = pytest.mark.gpu

PATHS = {
    "sector-default": {},
    "smem": {"FFQ_SECTOR": "0"},
    "graph-dense": {"FFQ_SMEM_MAX_QUBITS": "0", "FFQ_SUPPORT": "0", "FFQ_SECTOR": "0"},
    "graph-support": {"FFQ_SMEM_MAX_QUBITS": "0", "FFQ_SECTOR": "0"},
    "persistent": {"FFQ_SMEM_MAX_QUBITS": "0", "FFQ_PERSIST": "1", "FFQ_SECTOR": "0"},
    "sector": {"FFQ_SMEM_MAX_QUBITS": "0"},
}


def _ctx(monkeypatch, env):
    for k in ("FFQ_SMEM_MAX_QUBITS", "FFQ_SUPPORT", "FFQ_PERSIST", "FFQ_SECTOR", "FFQ_SECTOR_CL", "FFQ_SECTOR_REAL"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    return capi.Context(0)


def _oracle_state(oracle, n, hf, gens, theta):
    """gens: list of (x[], z[], c[]) per generator in execution order."""
    psi = oracle.hf_state(n, hf)
    for (x, z, c), t in zip(gens, theta):
        order = np.lexsort((z, x))  # canonical (x, z) order
        for i in order:
            psi = oracle.apply_pauli_rotation(n, psi, int(x[i]), int(z[i]), t * c[i].imag)
    return psi


def _plan_arrays(gens):
    off = [0]
    for g in gens:
        off.append(off[-1] + len(g[0]))
    x = np.concatenate([g[0] for g in gens]).astype(np.uint64)
    z = np.concatenate([g[1] for g in gens]).astype(np.uint64)
    c = np.concatenate([g[2] for g in gens])
    return np.array(off, np.int64), x, z, c


@pytest.mark.parametrize("path", list(PATHS))
def test_non_uccsd_generators_all_paths(monkeypatch, oracle, path):
    # generators that do not fuse: several flip masks, non-commuting strings
    n = 10
    rng = np.random.default_rng(7)
    gens = [
        (np.array([0b11, 0b1100]), np.array([0b10, 0b100]), np.array([0.3j, -0.2j])),  # two flip masks
        (np.array([1, 1]), np.array([0, 1]), np.array([0.25j, 0.4j])),  # X0 and Y0: anticommute
        (np.array([0b101 << 5]), np.array([0b111]), np.array([0.5j])),  # single string
    ]
    P = problems.config_problem(1)
    hx = rng.integers(0, 1 << n, 40).astype(np.uint64)
    hz = rng.integers(0, 1 << n, 40).astype(np.uint64)
    hc = rng.normal(size=40)
    theta = np.array([0.7, -1.1, 0.35])
    hf = 0b0000001111
    c = _ctx(monkeypatch, PATHS[path])
    plan = capi.Plan(c, n, *_plan_arrays(gens))
    assert plan.info() == (1, 4)  # the single-string generator fuses; the other two run string by string
    ham = capi.Hamiltonian(c, n, hx, hz, hc)
    e = capi.energy_batch(c, plan, ham, hf, theta[None, :])[0]
    psi = _oracle_state(oracle, n, hf, gens, theta)
    ref = oracle.expectation(n, psi, oracle.PauliSum.from_terms(n, hx, hz, hc)).real
    assert abs(e - ref) <= 1e-10
    st = capi.State(c, n, 1)
    st.set_basis(hf)
    st.apply_plan(plan, theta[None, :])
    assert np.abs(st.download()[0] - psi).max() <= 1e-12
    del P


def test_empty_batch_empty_hamiltonian_and_no_generators(ctx_default, oracle):
    c = ctx_default
    P = problems.config_problem(2)
    plan = capi.Plan(c, P.n_qubits, *P.plan_arrays())
    ham = capi.Hamiltonian(c, P.n_qubits, *P.ham_arrays())
    assert capi.energy_batch(c, plan, ham, P.hf, np.zeros((0, P.n_gen))).shape == (0,)
    empty = capi.Hamiltonian(c, P.n_qubits, np.zeros(0, np.uint64), np.zeros(0, np.uint64), np.zeros(0))
    assert capi.energy_batch(c, plan, empty, P.hf, P.plan_thetas())[0] == 0.0
    noplan = capi.Plan(c, P.n_qubits, np.zeros(1, np.int64), np.zeros(0, np.uint64), np.zeros(0, np.uint64),
                       np.zeros(0))
    e_hf = capi.energy_batch(c, noplan, ham, P.hf, np.zeros((1, 0)))[0]
    x, z, co = P.ham_arrays()
    ref = oracle.expectation(P.n_qubits, oracle.hf_state(P.n_qubits, P.hf),
                             oracle.PauliSum.from_terms(P.n_qubits, x, z, co)).real
    assert abs(e_hf - ref) <= 1e-12
    ident = capi.Hamiltonian(c, P.n_qubits, [0], [0], [2.5])
    assert abs(capi.energy_batch(c, plan, ident, P.hf, P.plan_thetas())[0] - 2.5) <= 1e-12  # norm 1


@pytest.fixture(scope="module")
def ctx_default():
    return capi.Context(0)


@pytest.mark.parametrize("config", [2, 3])
def test_theta_periodicity_and_zero(ctx_default, config):
    c = ctx_default
    P = problems.config_problem(config)
    plan = capi.Plan(c, P.n_qubits, *P.plan_arrays())
    ham = capi.Hamiltonian(c, P.n_qubits, *P.ham_arrays())
    th = P.plan_thetas()
    rows = np.vstack([th, th + 2 * np.pi, np.zeros_like(th)])
    e = capi.energy_batch(c, plan, ham, P.hf, rows)
    assert abs(e[0] - e[1]) <= 1e-10
    st = capi.State(c, P.n_qubits, 1)
    st.set_basis(P.hf)
    assert abs(e[2] - st.expectation(ham)[0].real) <= 1e-12


def test_batch_not_multiple_of_chunk(monkeypatch):
    # the graph path's last chunk recomputes stale rows; their outputs must not leak
    c = _ctx(monkeypatch, {"FFQ_SMEM_MAX_QUBITS": "0", "FFQ_SECTOR": "0"})
    monkeypatch.setenv("FFQ_SLAB_MB", "1")  # 1 MiB slab: 16 rows of 12 qubits per chunk
    c = capi.Context(0)
    P = problems.config_problem(2, batch=37)
    plan = capi.Plan(c, P.n_qubits, *P.plan_arrays())
    ham = capi.Hamiltonian(c, P.n_qubits, *P.ham_arrays())
    full = capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas())
    one = np.array([capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas()[i:i + 1])[0] for i in range(37)])
    assert np.array_equal(full, one)


def test_sector_single_cta_small_closure(monkeypatch, oracle):
    # 12 qubits: closure of 400 amplitudes -> the one-CTA sector kernel (default),
    # against the dense shared-memory evaluator (FFQ_SECTOR=0)
    P = problems.config_problem(2, batch=9)
    c = _ctx(monkeypatch, {})
    plan = capi.Plan(c, P.n_qubits, *P.plan_arrays())
    ham = capi.Hamiltonian(c, P.n_qubits, *P.ham_arrays())
    e = capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas())
    c2 = _ctx(monkeypatch, {"FFQ_SECTOR": "0"})
    plan2 = capi.Plan(c2, P.n_qubits, *P.plan_arrays())
    ham2 = capi.Hamiltonian(c2, P.n_qubits, *P.ham_arrays())
    assert np.abs(e - capi.energy_batch(c2, plan2, ham2, P.hf, P.plan_thetas())).max() <= 1e-12


@pytest.mark.parametrize("cl", ["4", "8"])
def test_sector_cluster_sizes_agree(monkeypatch, cl):
    # FFQ_SECTOR_CL is read per context: 2-CTA (default) vs 4- or 8-CTA clusters
    P = problems.config_problem(3, batch=3)
    e = {}
    for k in ("2", cl):
        c = _ctx(monkeypatch, {"FFQ_SECTOR_CL": k, "FFQ_SECTOR_REAL": "0"})
        plan, ham = capi.Plan(c, P.n_qubits, *P.plan_arrays()), capi.Hamiltonian(c, P.n_qubits, *P.ham_arrays())
        e[k] = capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas())
    assert np.abs(e[cl] - e["2"]).max() <= 1e-12


@pytest.mark.parametrize("env", [{}, {"FFQ_SECTOR": "0"}, {"FFQ_SMEM_MAX_QUBITS": "0", "FFQ_SECTOR": "0"}])
def test_reuploaded_hamiltonian_never_hits_stale_cache(monkeypatch, oracle, env):
    # plans cache compiled programs / captured graphs per Hamiltonian; a handle
    # destroyed and re-uploaded (often at the same address) must not reuse them
    c = _ctx(monkeypatch, env)
    P = problems.config_problem(2, batch=2)
    plan = capi.Plan(c, P.n_qubits, *P.plan_arrays())
    x, z, co = P.ham_arrays()
    rng = np.random.default_rng(11)
    for it in range(6):
        scale = 1.0 + it
        ham = capi.Hamiltonian(c, P.n_qubits, x, z, co * scale)
        e = capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas())
        if it == 0:
            base = e.copy()
        assert np.abs(e - base * scale).max() <= 1e-10 * scale
        del ham
    # a structurally different Hamiltonian (different groups) after the same churn
    hx = rng.integers(0, 1 << P.n_qubits, 30).astype(np.uint64)
    hz = rng.integers(0, 1 << P.n_qubits, 30).astype(np.uint64)
    hc = rng.normal(size=30)
    ham = capi.Hamiltonian(c, P.n_qubits, hx, hz, hc)
    e = capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas())
    hs = oracle.PauliSum.from_terms(P.n_qubits, hx, hz, hc)
    kind, idx = oracle.build_generators(P.n_qubits, P.n_elec)
    for b in range(2):
        ref, _ = oracle.energy_trotter(P.n_qubits, P.n_elec, kind, idx, np.array(P.plan.order, np.int32),
                                       P.thetas[b], hs)
        assert abs(e[b] - ref) <= 1e-10
    c2 = capi.Context(0)
    plan2 = capi.Plan(c2, P.n_qubits, *P.plan_arrays())
    ham2 = capi.Hamiltonian(c2, P.n_qubits, hx, hz, hc)
    assert np.abs(e - capi.energy_batch(c2, plan2, ham2, P.hf, P.plan_thetas())).max() <= 1e-12


@pytest.mark.parametrize("real", ["1", "0"])
def test_sector_info_config3(monkeypatch, real):
    P = problems.config_problem(3, batch=1)
    c = _ctx(monkeypatch, {"FFQ_SECTOR_REAL": real})
    plan, ham = capi.Plan(c, P.n_qubits, *P.plan_arrays()), capi.Hamiltonian(c, P.n_qubits, *P.ham_arrays())
    info = capi.sector_info(c, plan, ham, P.hf)
    # |S| = C(9,5)^2: the (5 alpha, 5 beta) sector of 9 spatial orbitals
    assert info["closure_size"] == 15876
    assert info["real_amplitudes"] == int(real)  # UCCSD F = +-1, real integrals
    assert info["ctas_per_eval"] == (1 if real == "1" else 2)
    assert (info["cluster_barrier_steps"] == 0) == (real == "1")
    assert info["cluster_barrier_steps"] <= P.n_gen
    assert info["expectation_rows"] * 32 + info["clique_pairs"] >= info["expectation_pairs"] > 0
    assert info["generator_pairs"] > 0
    # the real program lays S out as 126 alpha x 127 (odd stride) beta slots and
    # holds most expectation pairs in alpha-beta cliques (every alpha-beta pair:
    # 36 x 36 excitation masks x 35 x 70 pairs) and anchored string blocks
    assert info["slots"] == (126 * 127 if real == "1" else 15876)
    held = info["block_pairs"] + info["clique_pairs"]
    assert (held >= 0.8 * info["expectation_pairs"]) == (real == "1")
    assert info["clique_pairs"] == (36 * 36 * 35 * 70 if real == "1" else 0)
    if real == "1":  # the member order of the clique loads is bank-conflict free (model)
        assert info["clique_conflicts"] <= 4


def test_clique_expectation_matches_blocks(monkeypatch):
    """The alpha-beta cliques (alpha-first gauge, FFQ_CLIQUES=1, the default)
    against the anchored-block program without them (FFQ_CLIQUES=0) on config-3
    parameter-shift rows, including +-pi/2 shifts (oracle parity of the default
    program: tests/test_gpu_parity.py)."""
    from paper_2402_17993_b200 import parameter_shift_set

    P = problems.config_problem(3, batch=1)
    rows = np.array(parameter_shift_set(list(P.thetas[0]))).reshape(-1, P.n_gen)[::37]
    out = {}
    for cq in ("1", "0"):
        c = _ctx(monkeypatch, {"FFQ_CLIQUES": cq})
        plan, ham = capi.Plan(c, P.n_qubits, *P.plan_arrays()), capi.Hamiltonian(c, P.n_qubits, *P.ham_arrays())
        assert (capi.sector_info(c, plan, ham, P.hf)["clique_pairs"] > 0) == (cq == "1")
        out[cq] = capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas(rows))
        del plan, ham, c
    assert np.abs(out["1"] - out["0"]).max() <= 1e-12
    # and without the anchored blocks (every pair in the generic rows): 31 rows run
    # split over role warps, 3 of them alone on 8 CTAs each, as above
    monkeypatch.delenv("FFQ_CLIQUES", raising=False)
    c = _ctx(monkeypatch, {"FFQ_BLOCKS": "0"})
    plan, ham = capi.Plan(c, P.n_qubits, *P.plan_arrays()), capi.Hamiltonian(c, P.n_qubits, *P.ham_arrays())
    assert capi.sector_info(c, plan, ham, P.hf)["block_pairs"] == 0
    plain = capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas(rows))
    assert np.array_equal(plain[:3], capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas(rows[:3])))
    monkeypatch.delenv("FFQ_BLOCKS", raising=False)
    assert np.abs(out["1"] - plain).max() <= 1e-12


@pytest.mark.parametrize("config", [2, 3])
def test_real_amplitude_kernel_matches_complex(monkeypatch, oracle, config):
    # real F, real class sums, basis start: psi is real and the one-CTA
    # real-amplitude program must agree with the complex cluster program
    P = problems.config_problem(config, batch=6)
    out = {}
    for real in ("1", "0"):
        c = _ctx(monkeypatch, {"FFQ_SECTOR_REAL": real})
        plan, ham = capi.Plan(c, P.n_qubits, *P.plan_arrays()), capi.Hamiltonian(c, P.n_qubits, *P.ham_arrays())
        assert capi.sector_info(c, plan, ham, P.hf)["real_amplitudes"] == int(real)
        out[real] = capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas())
    assert np.abs(out["1"] - out["0"]).max() <= 1e-12
    kind, idx = oracle.build_generators(P.n_qubits, P.n_elec)
    x, z, co = P.ham_arrays()
    hs = oracle.PauliSum.from_terms(P.n_qubits, x, z, co)
    for b in range(2):
        ref, _ = oracle.energy_trotter(P.n_qubits, P.n_elec, kind, idx, np.array(P.plan.order, np.int32),
                                       P.thetas[b], hs)
        assert abs(out["1"][b] - ref) <= 1e-10


def test_complex_hamiltonian_takes_complex_program(monkeypatch):
    # a Hamiltonian with a non-real class sum (an XY-type string with real
    # coefficient gives an imaginary f) must not take the real-amplitude program
    P = problems.config_problem(2, batch=2)
    x, z, co = P.ham_arrays()
    x2 = np.concatenate([x, np.array([0b11], np.uint64)])
    z2 = np.concatenate([z, np.array([0b01], np.uint64)])  # Y0 X1
    c2 = np.concatenate([co, np.array([0.05])])
    c = _ctx(monkeypatch, {})
    plan, ham = capi.Plan(c, P.n_qubits, *P.plan_arrays()), capi.Hamiltonian(c, P.n_qubits, x2, z2, c2)
    assert capi.sector_info(c, plan, ham, P.hf)["real_amplitudes"] == 0
    e = capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas())
    c0 = _ctx(monkeypatch, {"FFQ_SECTOR": "0"})
    plan0, ham0 = capi.Plan(c0, P.n_qubits, *P.plan_arrays()), capi.Hamiltonian(c0, P.n_qubits, x2, z2, c2)
    assert np.abs(e - capi.energy_batch(c0, plan0, ham0, P.hf, P.plan_thetas())).max() <= 1e-12


def test_cli_energy_from_fcidump_and_vqe(tmp_path, capsys):
    """SPEC.md:578-629 CLI on the device: energies of a config read back from
    its FCIDUMP equal the config's own; the config-1 VQE converges below HF."""
    import json

    from paper_2402_17993_b200 import cli

    f = str(tmp_path / "c2.fcidump")
    assert cli.main(["ham", "--config", "2", "--out", f]) == 0
    capsys.readouterr()
    seed = problems.ham_seed(2)
    assert cli.main(["energy", "--fcidump", f, "--batch", "3", "--seed", str(seed)]) == 0
    rep = json.loads(capsys.readouterr().out)
    P = problems.config_problem(2, batch=3)
    c = capi.Context(0)
    ref = capi.energy_batch(c, capi.Plan(c, P.n_qubits, *P.plan_arrays()),
                            capi.Hamiltonian(c, P.n_qubits, *P.ham_arrays()), P.hf, P.plan_thetas())
    assert np.abs(np.array([r["total"] for r in rep["records"]]) - ref).max() <= 1e-10
    assert cli.main(["vqe", "--config", "1", "--optimizer", "bfgs"]) == 0
    r = json.loads(capsys.readouterr().out)["records"][0]
    assert r["converged"] and r["total"] < r["hf_energy"]
    # selftest: the CUDA path against the committed golden fixtures (no oracle import)
    assert cli.main(["selftest"]) == 0
    r = json.loads(capsys.readouterr().out)["records"][0]
    assert r["ok"] and r["max_energy_err"] <= 1e-10 and r["max_state_err"] <= 1e-12


def test_split_knob_bit_identical(monkeypatch):
    # FFQ_SPLIT caps the CTAs per 18-qubit evaluation (1 = one CTA each) and
    # FFQ_ROLES=0 turns the role warps off; the energies depend on neither.
    # Splits 4 / 8..32 run the block-stream segments on roles (0, 1, 1) / (1, 2, 3),
    # split 2 and the one-CTA program sum them on one warp (ffq_sector.cuh).
    P = problems.config_problem(3, batch=3)
    out = {}
    for split, roles in (("1", "1"), ("2", "1"), ("4", "1"), ("8", "1"), ("16", "1"), ("32", "1"), ("8", "0")):
        monkeypatch.delenv("FFQ_ROLES", raising=False)
        c = _ctx(monkeypatch, {"FFQ_SPLIT": split, "FFQ_ROLES": roles})
        plan = capi.Plan(c, P.n_qubits, *P.plan_arrays())
        ham = capi.Hamiltonian(c, P.n_qubits, *P.ham_arrays())
        out[split, roles] = capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas())
        del plan, ham, c
    for k, v in out.items():
        assert np.array_equal(out["1", "1"], v), k


@pytest.mark.parametrize("case", ["config5_20q", "uccsd_20q"])
def test_compact_sector_path_matches_dense(monkeypatch, case):
    # the compact real [alpha][beta] sector layout (ffq_compact.inl; the default
    # above 26 qubits) against the dense support-tracked path on the same inputs
    if case == "config5_20q":
        P = problems.config5_problem(n_doubles=300, n_terms=200, n_qubits=20, n_elec=10)
    else:
        P = problems.make_problem(10, 10, problems.ham_seed(9, 1), batch=2)
    out = {}
    for mode, env in (("compact", {"FFQ_COMPACT_MIN": "20"}), ("dense", {"FFQ_COMPACT": "0"})):
        for k in ("FFQ_COMPACT", "FFQ_COMPACT_MIN"):
            monkeypatch.delenv(k, raising=False)
        c = _ctx(monkeypatch, env)
        plan = capi.Plan(c, P.n_qubits, *P.plan_arrays())
        ham = capi.Hamiltonian(c, P.n_qubits, *P.ham_arrays())
        out[mode] = capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas())
        out[mode + "2"] = capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas())
        del plan, ham, c
    assert np.max(np.abs(out["compact"] - out["dense"])) <= 1e-10
    assert np.array_equal(out["compact"], out["compact2"])  # deterministic


@pytest.mark.parametrize("case", ["config5_20q", "uccsd_16q"])
def test_compact_interleaved_lanes_bit_identical(monkeypatch, case):
    # the compact layout evaluates 8, 4, 2 or 1 theta rows per matrix (lanes
    # interleaved per amplitude); a batch of 15 runs as 8 + 4 + 2 + 1 (9 as 8 + 1)
    # and must equal the one-row-at-a-time energies bit for bit (same pair order
    # per lane), and the dense support path to 1e-10
    if case == "config5_20q":
        P = problems.config5_problem(n_doubles=300, n_terms=200, n_qubits=20, n_elec=10)
        rng = np.random.default_rng(3)
        rows = np.concatenate([P.thetas, rng.uniform(-0.05, 0.05, size=(8, P.n_gen))])
    else:
        P = problems.make_problem(8, 8, problems.ham_seed(9, 2), batch=15)
        rows = P.thetas
    th = P.plan_thetas(rows)
    out = {}
    for mode, env in (("il8", {"FFQ_COMPACT_MIN": "0", "FFQ_SECTOR": "0"}),
                      ("il4", {"FFQ_COMPACT_MIN": "0", "FFQ_SECTOR": "0", "FFQ_COMPACT_IL": "4"}),
                      ("il1", {"FFQ_COMPACT_MIN": "0", "FFQ_SECTOR": "0", "FFQ_COMPACT_IL": "1"}),
                      ("dense", {"FFQ_COMPACT": "0", "FFQ_SECTOR": "0"})):
        for k in ("FFQ_COMPACT", "FFQ_COMPACT_MIN", "FFQ_COMPACT_IL", "FFQ_SECTOR"):
            monkeypatch.delenv(k, raising=False)
        c = _ctx(monkeypatch, env)
        plan = capi.Plan(c, P.n_qubits, *P.plan_arrays())
        ham = capi.Hamiltonian(c, P.n_qubits, *P.ham_arrays())
        n0 = c.launches()
        out[mode] = capi.energy_batch(c, plan, ham, P.hf, th)
        out[mode + "_launches"] = c.launches() - n0
        del plan, ham, c
    assert np.array_equal(out["il8"], out["il1"]) and np.array_equal(out["il4"], out["il1"])
    assert out["il8_launches"] < out["il4_launches"] < out["il1_launches"] // 2  # fewer matrix passes
    assert np.max(np.abs(out["il8"] - out["dense"])) <= 1e-10


def test_compact_sector_path_golden(monkeypatch):
    # the compact layout forced at configs 1-3 (FFQ_SECTOR=0 skips the closure
    # programs, FFQ_COMPACT_MIN=0 lets the compact path take every size) against
    # the committed oracle energies (tests/golden/energies.json)
    import json

    with open(os.path.join(os.path.dirname(__file__), "golden", "energies.json")) as f:
        golden = json.load(f)["configs"]
    monkeypatch.delenv("FFQ_COMPACT", raising=False)
    c = _ctx(monkeypatch, {"FFQ_SECTOR": "0", "FFQ_COMPACT_MIN": "0"})
    for cfg, g in golden.items():
        P = problems.config_problem(int(cfg), batch=len(g["rows"]))
        plan = capi.Plan(c, P.n_qubits, *P.plan_arrays())
        ham = capi.Hamiltonian(c, P.n_qubits, *P.ham_arrays())
        n0 = c.launches()
        e = capi.energy_batch(c, plan, ham, P.hf, P.plan_thetas())
        assert c.launches() - n0 > P.n_gen  # one pass per generator: the compact path ran
        ref = np.array([float.fromhex(r["energy"]) for r in g["rows"]])
        assert np.abs(e - ref).max() <= 1e-10, cfg


def test_sector_program_repeatable_under_load():
    """Evidence against shared-memory races in the barrier-pipelined real
    program (compute-sanitizer is closed on the GPU pool; the host check
    ffq_sector_emulate proves every generator step race-free by construction):
    ten launches of 300 config-3 rows, plus small batches that take the split
    path, give bit-identical energies."""
    P = problems.config_problem(3, batch=1)
    from paper_2402_17993_b200 import parameter_shift_set

    rows = np.array(parameter_shift_set(list(P.thetas[0]))).reshape(-1, P.n_gen)[:300]
    c = capi.Context(0)
    plan, ham = capi.Plan(c, P.n_qubits, *P.plan_arrays()), capi.Hamiltonian(c, P.n_qubits, *P.ham_arrays())
    th = P.plan_thetas(rows)
    ref = capi.energy_batch(c, plan, ham, P.hf, th)
    for _ in range(10):
        assert np.array_equal(capi.energy_batch(c, plan, ham, P.hf, th), ref)
    for nb in (1, 3, 17):
        assert np.array_equal(capi.energy_batch(c, plan, ham, P.hf, th[:nb]), ref[:nb])


def test_config5_full_size_conserved_quantities():
    """BASELINE config 5's plan at full size (32 qubits, 2128 generators) through
    the compact layout with Hamiltonians whose expectation is fixed by symmetry
    for every theta: the norm (H = I), the particle number (sum (I - Z_q) / 2 =
    16) and the alpha particle number (even qubits: 8). Size-independent checks
    of the generator passes at the size no oracle reaches."""
    import torch

    if torch.cuda.get_device_properties(0).total_memory < 40 * 2**30:
        pytest.skip("needs ~12 GiB of device memory")
    P = problems.config5_problem()
    c = capi.Context(0)
    plan = capi.Plan(c, 32, *P.plan_arrays())
    rng = np.random.default_rng(32)
    rows = np.concatenate([P.plan_thetas(), rng.uniform(-0.3, 0.3, size=(2, P.n_gen))])  # also larger angles

    def number_op(qubits):
        x = np.zeros(len(qubits) + 1, np.uint64)
        z = np.array([0] + [1 << q for q in qubits], np.uint64)
        co = np.array([0.5 * len(qubits)] + [-0.5] * len(qubits))
        return x, z, co

    for name, (x, z, co), want in (("norm", (np.zeros(1, np.uint64), np.zeros(1, np.uint64), np.ones(1)), 1.0),
                                   ("N", number_op(range(32)), 16.0),
                                   ("N_alpha", number_op(range(0, 32, 2)), 8.0)):
        ham = capi.Hamiltonian(c, 32, x, z, co)
        e = capi.energy_batch(c, plan, ham, P.hf, rows)
        assert np.abs(e - want).max() <= 1e-10, (name, e)
        del ham


def test_expectation_is_linear_in_the_hamiltonian_18q():
    """<psi|H|psi> is linear in H: the 9316-term config-3 Hamiltonian split at
    random into two halves (neither is molecular: their alpha-beta weights need
    not factorise, so the clique check may refuse groups and the anchored blocks
    or generic rows take them) must add up to the full energy on +-pi/2 shift
    rows. Exercises the fallbacks of the expectation compiler at 18 qubits."""
    from paper_2402_17993_b200 import parameter_shift_set

    P = problems.config_problem(3, batch=1)
    rows = np.array(parameter_shift_set(list(P.thetas[0]))).reshape(-1, P.n_gen)[::97]
    th = P.plan_thetas(rows)
    c = capi.Context(0)
    plan = capi.Plan(c, P.n_qubits, *P.plan_arrays())
    x, z, co = P.ham_arrays()
    pick = np.random.default_rng(18).random(len(x)) < 0.5
    full = capi.energy_batch(c, plan, capi.Hamiltonian(c, P.n_qubits, x, z, co), P.hf, th)
    parts = []
    for m in (pick, ~pick):
        ham = capi.Hamiltonian(c, P.n_qubits, x[m], z[m], co[m])
        parts.append(capi.energy_batch(c, plan, ham, P.hf, th))
        info = capi.sector_info(c, plan, ham, P.hf)
        assert info["real_amplitudes"] == 1 and info["expectation_pairs"] > 0
        del ham
    assert np.abs(parts[0] + parts[1] - full).max() <= 1e-10


def test_energy_batch_pinned_and_pageable_inputs_agree(ctx_default):
    """ffq_energy_batch reads theta in place when it lies in page-locked host
    memory and stages it through its own pinned buffer otherwise; large batches
    go in chunks of SM waves. Same energies bit for bit either way."""
    import torch

    from paper_2402_17993_b200 import parameter_shift_set

    c = ctx_default
    P = problems.config_problem(3, batch=1)
    rows = np.array(parameter_shift_set(list(P.thetas[0]))).reshape(-1, P.n_gen)[:400]  # 1.8 MB: the chunked path
    th = P.plan_thetas(rows)
    plan = capi.Plan(c, P.n_qubits, *P.plan_arrays())
    ham = capi.Hamiltonian(c, P.n_qubits, *P.ham_arrays())
    pinned = torch.from_numpy(th).pin_memory().numpy()
    a = capi.energy_batch(c, plan, ham, P.hf, th)
    b = capi.energy_batch(c, plan, ham, P.hf, pinned)
    assert np.array_equal(a, b)
    assert np.array_equal(a[:3], capi.energy_batch(c, plan, ham, P.hf, pinned[:3]))  # unchunked
