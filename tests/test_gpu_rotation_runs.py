"""GPU parity of ffq_state_apply_pauli_rotations: runs of rotations whose flip
masks lie in the low 12 qubits are applied per TMA-staged shared-memory tile
(k_rotation_run, one HBM round trip per run), the others one pass each
(k_pauli_rotation). Checked through the C-ABI against the oracle's
apply_pauli_rotation string by string, against the unfused
path (FFQ_ROT_TILE=0), and at 26 qubits through run-then-inverse-run.

Tolerance: amplitudes <= 1e-12 max-abs (north_star)."""
import numpy as np
import pytest

from paper_2402_17993_b200 import capi

pytestmark = pytest.mark.gpu

A_TOL = 1e-12


@pytest.fixture(scope="module")
def ctx():
    return capi.Context(0)


def random_state(rng, n, batch):
    psi = rng.normal(size=(batch, 1 << n)) + 1j * rng.normal(size=(batch, 1 << n))
    return psi / np.linalg.norm(psi, axis=1, keepdims=True)


def random_strings(rng, n, count, low_frac=0.7):
    """Mixed list: low flip masks (x < 2^min(n,12), incl. x = 0 and x odd),
    high flip masks, z anywhere."""
    lo = min(n, 12)
    x = np.zeros(count, np.uint64)
    z = rng.integers(0, 1 << n, size=count, dtype=np.uint64)
    for r in range(count):
        u = rng.random()
        if u < 0.1:
            x[r] = 0
        elif u < low_frac:
            x[r] = rng.integers(1, 1 << lo)
        else:
            x[r] = rng.integers(1, 1 << n)
    th = rng.uniform(-np.pi, np.pi, size=count)
    return x, z, th


@pytest.mark.parametrize("n", [2, 5, 11, 12, 13, 16])
def test_rotation_runs_vs_oracle(ctx, oracle, n):
    rng = np.random.default_rng(100 + n)
    psi = random_state(rng, n, 2)
    x, z, th = random_strings(rng, n, 48)
    st = capi.State(ctx, n, 2)
    st.upload(psi)
    st.rotate_many(x, z, th)
    ref = psi.copy()
    for b in range(2):
        for r in range(len(x)):
            ref[b] = oracle.apply_pauli_rotation(n, ref[b], int(x[r]), int(z[r]), float(th[r]))
    assert np.abs(st.download() - ref).max() <= A_TOL


@pytest.mark.parametrize("high", [False, True])
def test_fused_runs_equal_unfused_and_launch_count(monkeypatch, high):
    """One run of 32 rotations: flip masks in the low 12 qubits (TMA tile) or on
    qubits 0-4 and 13-19 (gathered tile), batch of 3 rows."""
    n = 20
    rng = np.random.default_rng(7 + high)
    psi = random_state(rng, n, 3)
    x = rng.integers(1, 1 << 12, size=32, dtype=np.uint64)
    if high:
        x = np.array([(int(v) & 31) | ((int(v) >> 5) << (n - 7)) for v in x], np.uint64)
    z = rng.integers(0, 1 << n, size=32, dtype=np.uint64)
    th = rng.uniform(-1, 1, size=32)
    out = {}
    for tile in ("12", "0"):
        monkeypatch.setenv("FFQ_ROT_TILE", tile)
        c = capi.Context(0)
        st = capi.State(c, n, 3)
        st.upload(psi)
        l0 = c.launches()
        st.rotate_many(x, z, th)
        out[tile] = (st.download(), c.launches() - l0)
        del st  # the state before its context
        c.close()
    assert out["12"][1] == 1 and out["0"][1] == 32
    assert np.abs(out["12"][0] - out["0"][0]).max() <= 1e-14


def test_rotation_run_inverse_roundtrip_26q(ctx):
    # 26 qubits (1 GiB): a mixed run, then the inverse run (reverse order, -theta) = I
    n = 26
    rng = np.random.default_rng(3)
    psi = (rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)) / np.sqrt(2 << n)
    x, z, th = random_strings(rng, n, 24)
    st = capi.State(ctx, n, 1)
    st.upload(psi)
    st.rotate_many(x, z, th)
    mid = st.download()[0]
    assert abs(np.linalg.norm(mid) - np.linalg.norm(psi)) <= 1e-12
    st.rotate_many(x[::-1].copy(), z[::-1].copy(), -th[::-1])
    assert np.abs(st.download()[0] - psi).max() <= A_TOL


def test_rotation_runs_edges(ctx):
    st = capi.State(ctx, 6, 1)
    st.set_basis(5)
    st.rotate_many(np.zeros(0, np.uint64), np.zeros(0, np.uint64), np.zeros(0))  # empty list: no-op
    assert st.download()[0][5] == 1.0
    with pytest.raises(Exception):
        st.rotate_many(np.array([1 << 6], np.uint64), np.array([0], np.uint64), np.array([0.1]))
    with pytest.raises(capi.ContractViolation):
        st.rotate_many(np.array([1, 2], np.uint64), np.array([0], np.uint64), np.array([0.1]))


def test_plan_string_runs_fused_equal_unfused(monkeypatch):
    """Plan path (run_plan_ops): consecutive string ops with low flip masks run
    as one k_rotation_run inside the captured graph. SCBKT config 3 (16 qubits,
    every generator as per-string rotations): energies equal the unfused
    passes' to 1e-12 with fewer launches; the JW energies are the anchor
    (test_scbkt_energies_match_jw)."""
    from paper_2402_17993_b200 import problems

    R = problems.config_problem(3, batch=2, mapping="scbkt")
    J = problems.config_problem(3, batch=2)
    res = {}
    for tile in ("12", "0"):
        monkeypatch.setenv("FFQ_ROT_TILE", tile)
        c = capi.Context(0)
        plan = capi.Plan(c, R.n_qubits, *R.plan_arrays())
        ham = capi.Hamiltonian(c, R.n_qubits, *R.ham_arrays())
        l0 = c.launches()
        e = capi.energy_batch(c, plan, ham, R.hf, R.plan_thetas())
        res[tile] = (e, c.launches() - l0)
        del plan, ham
        c.close()
    assert np.abs(res["12"][0] - res["0"][0]).max() <= 1e-12
    assert res["12"][1] < res["0"][1]
    c = capi.Context(0)
    plan = capi.Plan(c, J.n_qubits, *J.plan_arrays())
    ham = capi.Hamiltonian(c, J.n_qubits, *J.ham_arrays())
    ej = capi.energy_batch(c, plan, ham, J.hf, J.plan_thetas())
    del plan, ham
    c.close()
    assert np.abs(res["12"][0] - ej).max() <= 1e-10


@pytest.mark.parametrize("n", [14, 17])
def test_gathered_tile_runs_vs_oracle_deterministic(ctx, oracle, n):
    """The gathered-tile path of k_rotation_run (a run's qubit set is not the
    low 12: flip masks on qubits 0-4 plus high qubits) against the oracle,
    deterministically: every run here needs gathered tiles, z spans all qubits,
    batch of 3."""
    rng = np.random.default_rng(1000 + n)
    psi = random_state(rng, n, 3)
    hi = [n - 1, n - 3, n - 6]
    xs = []
    for r in range(24):
        low = int(rng.integers(0, 32))
        high = sum(1 << q for q in hi if rng.random() < 0.6) or (1 << hi[r % 3])
        xs.append(low | high)
    x = np.array(xs, np.uint64)
    z = rng.integers(0, 1 << n, size=len(x), dtype=np.uint64)
    th = rng.uniform(-np.pi, np.pi, size=len(x))
    run_of, _, _, run_q, _, _ = capi.rotation_groups(n, 12, x)
    assert (run_of >= 0).all()  # every rotation runs fused
    low12 = (1 << 12) - 1
    assert all(int(q) & ~low12 for q in run_q)  # and every run gathers (its qubit set is not the low 12)
    st = capi.State(ctx, n, 3)
    st.upload(psi)
    l0 = ctx.launches()
    st.rotate_many(x, z, th)
    assert ctx.launches() - l0 < len(x)
    ref = psi.copy()
    for b in range(3):
        for r in range(len(x)):
            ref[b] = oracle.apply_pauli_rotation(n, ref[b], int(x[r]), int(z[r]), float(th[r]))
    assert np.abs(st.download() - ref).max() <= A_TOL
