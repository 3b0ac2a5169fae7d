"""Sharded state (a15): 2^g ranks emulated on one device through the same
pack/unpack exchange kernels the NCCL transport uses; energies and amplitudes
must match the unsharded path. The NCCL transport itself runs with world = 1
here (one GPU per gpurun call)."""
import numpy as np
import pytest

from paper_2402_17993_b200 import capi, problems

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return capi.Context(0)


@pytest.mark.parametrize("config,g", [(2, 1), (2, 2), (2, 3), (3, 2)])
def test_sharded_energy_and_state_match_unsharded(ctx, config, g):
    P = problems.config_problem(config)
    plan = capi.Plan(ctx, P.n_qubits, *P.plan_arrays())
    ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
    th = P.plan_thetas()[0]
    sh = capi.ShardedState(ctx, P.n_qubits, g)
    e = sh.energy(plan, ham, P.hf, th)
    e_ref = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())[0]
    assert abs(e - e_ref) <= 1e-12
    st = capi.State(ctx, P.n_qubits, 1)
    st.set_basis(P.hf)
    st.apply_plan(plan, P.plan_thetas())
    assert np.abs(sh.download() - st.download()[0]).max() <= 1e-12
    swaps, perm = sh.info()
    assert sorted(perm.tolist()) == list(range(P.n_qubits))
    assert (swaps > 0) == (g > 0)


def test_sharded_random_pauli_hamiltonian(ctx, oracle):
    # config-5-style H (random {I,X,Y,Z} strings: generic x-groups) at 14 qubits
    import paper_2402_17993_b200 as ff

    P = problems.make_problem(7, 6, problems.ham_seed(5), name="c5small")
    H = ff.random_pauli_hamiltonian(14, 300, problems.ham_seed(5) + 7)
    x, z, c = H.arrays()
    plan = capi.Plan(ctx, 14, *P.plan_arrays())
    ham = capi.Hamiltonian(ctx, 14, x, z, c)
    th = P.plan_thetas()[0]
    e1 = capi.ShardedState(ctx, 14, 0).energy(plan, ham, P.hf, th)
    e3 = capi.ShardedState(ctx, 14, 3).energy(plan, ham, P.hf, th)
    kind, idx = oracle.build_generators(14, 6)
    ref = oracle.energy_trotter(14, 6, kind, idx, np.array(P.plan.order, np.int32), P.thetas[0],
                                oracle.PauliSum.from_terms(14, x, z, c))[0]
    assert abs(e1 - ref) <= 1e-10 and abs(e3 - ref) <= 1e-10


def test_nccl_transport_world_one(ctx):
    P = problems.config_problem(2)
    plan = capi.Plan(ctx, P.n_qubits, *P.plan_arrays())
    ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
    sh = capi.ShardedState(ctx, P.n_qubits, 0, rank=0, nccl_id=capi.nccl_unique_id())
    e = sh.energy(plan, ham, P.hf, P.plan_thetas()[0])
    assert abs(e - capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())[0]) <= 1e-12


def test_config5_structure_small_vs_oracle(ctx, oracle):
    # config 5 recipe (singles + first doubles, random Pauli H) at 16 qubits,
    # through both the support-tracked graph path and the sharded path
    P = problems.config5_problem(n_doubles=150, n_terms=400, n_qubits=16, n_elec=8)
    x, z, c = P.ham_arrays()
    plan = capi.Plan(ctx, 16, *P.plan_arrays())
    ham = capi.Hamiltonian(ctx, 16, x, z, c)
    e = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())[0]
    e_sh = capi.ShardedState(ctx, 16, 2).energy(plan, ham, P.hf, P.plan_thetas()[0])
    psi = oracle.hf_state(16, P.hf)
    for gid in P.plan.order:
        gx, gz, gc = P.gens[gid].image.arrays()
        for xx, zz, cc in zip(gx, gz, gc):
            psi = oracle.apply_pauli_rotation(16, psi, int(xx), int(zz), P.thetas[0][gid] * cc.imag)
    ref = oracle.expectation(16, psi, oracle.PauliSum.from_terms(16, x, z, c)).real
    assert abs(e - ref) <= 1e-10 and abs(e_sh - ref) <= 1e-10


def test_dense_and_support_tracked_shard_paths_agree(monkeypatch):
    """The sharded path keeps a support bitmap per shard (support-tracked
    generator passes, expectation batched over the bitmaps, swaps that move
    (index, value) lists); FFQ_SUPPORT=0 selects the dense passes and dense
    half-shard swaps. Both run the config-5 recipe at 16 qubits on 3 global
    qubits and must agree in energy and amplitudes; the tracked path repeats
    bit for bit (its swap lists are filled in arbitrary order)."""
    P = problems.config5_problem(n_doubles=150, n_terms=400, n_qubits=16, n_elec=8)
    th = P.plan_thetas()[0]
    out = {}
    for mode, env in (("tracked", {}), ("dense", {"FFQ_SUPPORT": "0"})):
        monkeypatch.delenv("FFQ_SUPPORT", raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        c = capi.Context(0)
        plan = capi.Plan(c, 16, *P.plan_arrays())
        ham = capi.Hamiltonian(c, 16, *P.ham_arrays())
        sh = capi.ShardedState(c, 16, 3)
        e1 = sh.energy(plan, ham, P.hf, th)
        psi = sh.download().copy()
        e2 = sh.energy(plan, ham, P.hf, th)
        assert e1 == e2 and np.array_equal(psi, sh.download())
        out[mode] = (e1, psi, sh.info()[0])
        del sh, plan, ham, c
    monkeypatch.delenv("FFQ_SUPPORT", raising=False)
    assert abs(out["tracked"][0] - out["dense"][0]) <= 1e-12
    assert np.abs(out["tracked"][1] - out["dense"][1]).max() <= 1e-12
    assert out["tracked"][2] == out["dense"][2] > 0  # same swap schedule


def test_config5_full_size_sharded_equals_compact():
    """BASELINE config 5 at its full size (32 qubits, 16 electrons, 2128
    generators, 5000 Pauli terms): the sharded complex128 state on 3 global
    qubits (8 shards of 8 GiB emulated on this device with the NCCL path's
    kernels, 172 swaps) against the compact real sector layout (1.3 GB). Two
    implementations that share only the plan and Hamiltonian compilers must
    agree to 1e-10 Hartree; a zero-amplitude row must give <HF|H|HF>, which is
    exactly 0 for this Hamiltonian (no term is diagonal)."""
    import torch

    if torch.cuda.get_device_properties(0).total_memory < 120 * 2**30:
        pytest.skip("needs ~80 GiB of device memory")
    P = problems.config5_problem()
    c = capi.Context(0)
    plan = capi.Plan(c, 32, *P.plan_arrays())
    ham = capi.Hamiltonian(c, 32, *P.ham_arrays())
    x, _, _ = P.ham_arrays()
    assert int((np.asarray(x) == 0).sum()) == 0
    rows = np.concatenate([P.plan_thetas(), np.zeros((1, P.n_gen))])
    e_compact = capi.energy_batch(c, plan, ham, P.hf, rows)
    assert e_compact[1] == 0.0
    sh = capi.ShardedState(c, 32, 3)
    e_sh = sh.energy(plan, ham, P.hf, rows[0])
    swaps, perm = sh.info()
    del sh
    assert swaps > 100 and sorted(perm.tolist()) == list(range(32))
    assert abs(e_sh - e_compact[0]) <= 1e-10


@pytest.mark.parametrize("cfg,n", [(1, 8), (2, 12)])
def test_every_shard_size_with_random_pauli_hamiltonian(ctx, cfg, n):
    """Every global-qubit count the plan allows (a double needs 4 local qubits),
    with a random-string Hamiltonian (generic one-term groups): covers shards of
    16 amplitudes (no bitmap path), 32 (one-word bitmaps), 64 and more
    (support-tracked passes and support-compacted swaps)."""
    import paper_2402_17993_b200 as ff

    P = problems.config_problem(cfg)
    x, z, co = ff.random_pauli_hamiltonian(n, 200, 77 + cfg).arrays()
    plan = capi.Plan(ctx, n, *P.plan_arrays())
    ham = capi.Hamiltonian(ctx, n, x, z, co)
    ref = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())[0]
    for g in range(0, min(6, n - 4) + 1):
        e = capi.ShardedState(ctx, n, g).energy(plan, ham, P.hf, P.plan_thetas()[0])
        assert abs(e - ref) <= 1e-12, (g, e, ref)
    # fewer than 4 local qubits (n = 8) or more than 6 global ones (n = 12): refused, not a wrong number
    with pytest.raises(Exception):
        capi.ShardedState(ctx, n, n - 3).energy(plan, ham, P.hf, P.plan_thetas()[0])
