"""World-size-2 gloo tests on CPU of the multi-GPU host path: fragment
sharding by cost, row sharding, and the fixed-order gather + FMO assembly.
The per-unit compute is the CPU oracle here (no device in this container)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2402_17993_b200 as ff
from paper_2402_17993_b200 import dist as fdist, problems


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _small_fragments():
    frags, probs = [], {}
    for f in (1, 2, 3):
        probs[str(f)] = problems.make_problem(2, 2, problems.ham_seed(4, f), name=f"m{f}")
    for k, lab in enumerate(("21", "31", "32")):
        probs[lab] = problems.make_problem(3, 4, problems.ham_seed(4, 10 + k), name=f"d{lab}")
    for lab, P in probs.items():
        frags.append(ff.FragmentProblem(lab, P.H, P.plan, P.hf, list(P.thetas[0])))
    return frags, probs


def _oracle_eval(probs):
    from oracle import ffo

    def evaluate(fragments, rank, world):
        owner = fdist.fragment_owners(fragments, world)
        out = {}
        for f, o in zip(fragments, owner):
            if o != rank:
                continue
            P = probs[f.label]
            x, z, c = P.ham_arrays()
            H = ffo.PauliSum.from_terms(P.n_qubits, x, z, c)
            kind, idx = ffo.build_generators(P.n_qubits, P.n_elec)
            out[f.label] = ffo.energy_trotter(P.n_qubits, P.n_elec, kind, idx, np.array(P.plan.order, np.int32),
                                              P.thetas[0], H)[0]
        return out

    return evaluate


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        frags, probs = _small_fragments()
        e, energies = fdist.fmo_energy(frags, 3, _oracle_eval(probs))
        lo, hi = fdist.row_range(10, rank, world)
        rows = fdist.gather_rows(np.arange(lo, hi, dtype=np.float64) * 0.5, 10)
        q.put((rank, e, energies, rows.tolist()))
    finally:
        dist.destroy_process_group()


def test_fmo_and_rows_sharded_over_two_ranks():
    frags, probs = _small_fragments()
    e1 = ff.assemble_fragments(3, _oracle_eval(probs)(frags, 0, 1))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, e, energies, rows in res:
        assert e == e1  # bitwise: same per-unit compute, fixed assembly order
        assert sorted(energies) == ["1", "2", "21", "3", "31", "32"]
        assert rows == [0.5 * i for i in range(10)]


def _rows_worker(rank, world, port, q):
    """One config-1 parameter-shift set split over the ranks by the product's
    dist.row_range; each rank evaluates its block (oracle compute: no device
    here), dist.gather_rows reassembles it in rank order."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ffo

        ffo.set_threads(1)  # ranks share the host cores (OpenMP would oversubscribe)
        P = problems.config_problem(1)
        rows = np.array(ff.parameter_shift_set(list(P.thetas[0]))).reshape(-1, P.n_gen)
        lo, hi = fdist.row_range(rows.shape[0], rank, world)
        H = ffo.PauliSum.from_terms(P.n_qubits, *P.ham_arrays())
        kind, idx = ffo.build_generators(P.n_qubits, P.n_elec)
        order = np.array(P.plan.order, np.int32)
        mine = [ffo.energy_trotter(P.n_qubits, P.n_elec, kind, idx, order, rows[r], H)[0] for r in range(lo, hi)]
        q.put((rank, fdist.gather_rows(np.array(mine), rows.shape[0]).tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gradient_rows_split_over_ranks_bitwise(world):
    from oracle import ffo

    P = problems.config_problem(1)
    rows = np.array(ff.parameter_shift_set(list(P.thetas[0]))).reshape(-1, P.n_gen)
    H = ffo.PauliSum.from_terms(P.n_qubits, *P.ham_arrays())
    kind, idx = ffo.build_generators(P.n_qubits, P.n_elec)
    order = np.array(P.plan.order, np.int32)
    full = [ffo.energy_trotter(P.n_qubits, P.n_elec, kind, idx, order, r, H)[0] for r in rows]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rows_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, got in res:
        assert got == full  # bitwise, in row order, on every rank


def test_shard_by_cost_is_balanced_and_deterministic():
    costs = [1.0, 1.0, 1.0, 300.0, 300.0, 300.0]
    assert ff.shard_by_cost(costs, 1) == [0] * 6
    own = ff.shard_by_cost(costs, 3)
    assert sorted(own[3:]) == [0, 1, 2]  # the three dimers land on distinct ranks
    assert own == ff.shard_by_cost(costs, 3)
    assert [fdist.row_range(10, r, 3) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
    with pytest.raises(ff.ContractViolation):
        ff.shard_by_cost(costs, 0)
