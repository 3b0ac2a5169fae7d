"""Config 4 (FMO fragment batch) on the GPU through the C++ facade:
3 monomers at 12 qubits + 3 dimers at 18 qubits, assembled with the
reference's two-body formula (fmo.cpp:28-48)."""
import numpy as np
import pytest

import paper_2402_17993_b200 as ff
from paper_2402_17993_b200 import problems

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fmo():
    dev = ff.Device(0)
    frags = problems.fmo_fragment_problems()
    return dev, frags, ff.evaluate_fragments(dev, frags)


def test_fmo_fragments_vs_oracle(fmo, oracle):
    dev, frags, energies = fmo
    probs = problems.fmo_fragments()
    for lab in ("1", "2", "3", "21"):
        P = probs[lab]
        x, z, c = P.ham_arrays()
        H = oracle.PauliSum.from_terms(P.n_qubits, x, z, c)
        kind, idx = oracle.build_generators(P.n_qubits, P.n_elec)
        ref = oracle.energy_trotter(P.n_qubits, P.n_elec, kind, idx, np.array(P.plan.order, np.int32),
                                    P.thetas[0], H)[0]
        assert abs(energies[lab] - ref) <= 1e-10, lab


def test_fmo_sharded_equals_single_and_assembles(fmo):
    dev, frags, energies = fmo
    for world in (2, 4, 8):
        union = {}
        for r in range(world):
            part = ff.evaluate_fragments(dev, frags, r, world)
            assert not (set(part) & set(union))
            union.update(part)
        assert union == energies  # bitwise: same device path per fragment
    e = ff.assemble_fragments(3, energies)
    mono = sum(energies[k] for k in ("1", "2", "3"))
    dim = sum(energies[k] for k in ("21", "31", "32"))
    assert abs(e - (dim - mono)) <= 1e-12  # N_f = 3: E = sum E_IJ - sum E_I
    fmo2 = mono + sum(energies[a + b] - energies[a] - energies[b] for a, b in (("2", "1"), ("3", "1"), ("3", "2")))
    assert abs(e - fmo2) <= 1e-10  # FMO2 form (BASELINE.json config 4)


def test_multi_capi_equals_one_context_bitwise():
    """ffq_multi_* (one host thread per device, rows / units sharded, no
    collective) on the devices of this box against one context: the config-3
    gradient rows (ffq_multi_energy_batch) and the config-4 fragments' shift
    sets (ffq_multi_energy_units, assigned by cost) are bit-identical."""
    import paper_2402_17993_b200 as ff
    from paper_2402_17993_b200 import capi, problems

    n_dev = ff.Device.count()
    m = capi.Multi(list(range(n_dev)))
    assert m.device_count() == n_dev
    P = problems.config_problem(3)
    rows = np.array(ff.parameter_shift_set(list(P.thetas[0]))).reshape(-1, P.n_gen)[:300]
    pid = m.upload(P.n_qubits, P.plan_arrays(), P.ham_arrays())
    e_multi = m.energy_batch(pid, P.hf, P.plan_thetas(rows))
    ctx = capi.Context(0)
    plan = capi.Plan(ctx, P.n_qubits, *P.plan_arrays())
    ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
    assert np.array_equal(e_multi, capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas(rows)))
    frs = list(problems.fmo_fragments().values())
    pids = [m.upload(F.n_qubits, F.plan_arrays(), F.ham_arrays()) for F in frs]
    ths = [F.plan_thetas(np.array(ff.parameter_shift_set(list(F.thetas[0]))).reshape(-1, F.n_gen)[:40]) for F in frs]
    es, devs = m.energy_units(pids, [F.hf for F in frs], ths)
    assert all(0 <= d < n_dev for d in devs)
    for F, th, e in zip(frs, ths, es):
        pl = capi.Plan(ctx, F.n_qubits, *F.plan_arrays())
        hm = capi.Hamiltonian(ctx, F.n_qubits, *F.ham_arrays())
        assert np.array_equal(e, capi.energy_batch(ctx, pl, hm, F.hf, th))
    with pytest.raises(ff.ContractViolation):
        capi.Multi([0, 0])


def test_energy_prepare_concurrent_compile_equals_lazy_compile():
    """ffq_energy_prepare compiles the device program ahead of the first energy
    call and is re-entrant for distinct plans of one context: three fragments
    prepared from three host threads give the energies of the lazily compiled
    programs bit for bit, and the first energy call no longer pays the compile."""
    import threading
    import time

    import numpy as np

    from paper_2402_17993_b200 import capi, problems

    frs = [problems.make_problem(9, 10, problems.ham_seed(4, 10 + k)) for k in range(2)]
    frs.append(problems.make_problem(6, 6, problems.ham_seed(4, 1)))
    lazy = []
    c0 = capi.Context(0)
    for P in frs:
        plan = capi.Plan(c0, P.n_qubits, *P.plan_arrays())
        ham = capi.Hamiltonian(c0, P.n_qubits, *P.ham_arrays())
        lazy.append(capi.energy_batch(c0, plan, ham, P.hf, P.plan_thetas()))
        del plan, ham
    c1 = capi.Context(0)
    hs = [(capi.Plan(c1, P.n_qubits, *P.plan_arrays()), capi.Hamiltonian(c1, P.n_qubits, *P.ham_arrays())) for P in frs]
    errs = []

    def work(k):
        try:
            capi.energy_prepare(c1, hs[k][0], hs[k][1], frs[k].hf)
        except Exception as ex:  # surfaced below
            errs.append(ex)

    ts = [threading.Thread(target=work, args=(k,)) for k in range(len(frs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    t0 = time.perf_counter()
    eager = [capi.energy_batch(c1, hs[k][0], hs[k][1], frs[k].hf, frs[k].plan_thetas()) for k in range(len(frs))]
    first_calls_s = time.perf_counter() - t0
    for a, b in zip(lazy, eager):
        assert np.array_equal(a, b)
    assert first_calls_s < 0.5  # three evaluations without a compile
