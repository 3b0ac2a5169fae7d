"""Sharded state across real processes (gloo, CPU): the swap schedule of the
C-ABI (ffq_shard_schedule_steps), the half-shard pack/unpack index math of
k_swap_pack/k_swap_unpack (and of the support-compacted swap: counts first,
then (index, value) lists) and the per-pattern partner exchange of the sharded
expectation, executed by 2 and 4 ranks with torch.distributed point-to-point
messages. The per-shard compute is the CPU oracle (no device here); energies
and the gathered logical state must equal the unsharded oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2402_17993_b200 import capi, problems


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _permute(m, perm):
    r = 0
    for q, pq in enumerate(perm):
        if (m >> q) & 1:
            r |= 1 << int(pq)
    return r


def _exchange(buf, partner):
    out = torch.empty_like(buf)
    ops = [dist.P2POp(dist.isend, buf, partner), dist.P2POp(dist.irecv, out, partner)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    return out


def _exchange_lists(idx, vals, partner):
    """The support-compacted swap's wire protocol (shard_swap_sparse): the two
    counts first (one int64 each way), then `count` indices and values each way."""
    n_mine = torch.tensor([len(idx)], dtype=torch.int64)
    n_peer = int(_exchange(n_mine, partner)[0])
    r_idx = torch.empty(n_peer, dtype=torch.int64)
    r_val = torch.empty(n_peer, dtype=torch.complex128)
    ops = []
    if len(idx):
        ops += [dist.P2POp(dist.isend, torch.from_numpy(idx), partner),
                dist.P2POp(dist.isend, torch.from_numpy(vals), partner)]
    if n_peer:
        ops += [dist.P2POp(dist.irecv, r_idx, partner), dist.P2POp(dist.irecv, r_val, partner)]
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    return r_idx.numpy(), r_val.numpy()


def _half_indices(l, lpos, val):
    """k_swap_pack order: u ascending, zero inserted at lpos, bit lpos = val."""
    u = np.arange(1 << (l - 1), dtype=np.int64)
    lo = u & ((1 << lpos) - 1)
    return ((u >> lpos) << (lpos + 1)) | lo | (val << lpos)


def _worker(rank, world, port, q, n, ne, seed, sparse=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ffo

        g = world.bit_length() - 1
        l = n - g
        P = problems.make_problem(n // 2, ne, seed)
        off, x, z, c = P.plan_arrays()
        ip, fp, steps = capi.shard_schedule_steps(n, g, off, x, z, c)
        perm = ip.astype(np.int64).copy()
        shard = np.zeros(1 << l, complex)
        hfp = _permute(P.hf, perm)
        if hfp >> l == rank:
            shard[hfp & ((1 << l) - 1)] = 1.0
        theta = P.plan_thetas()[0]
        mask = (1 << l) - 1
        for kind, gpos, lpos, gen in steps:
            if kind == 0:  # swap physical global position gpos with local lpos
                j = gpos - l
                bit = (rank >> j) & 1
                idx = _half_indices(l, int(lpos), 1 - bit)
                if sparse:
                    # k_swap_pack_sparse / k_swap_unpack_sparse: only the non-zero amplitudes of the half
                    # move, as (index within the half, value); the slots they leave are cleared
                    u = np.nonzero(shard[idx] != 0)[0].astype(np.int64)
                    vals = np.ascontiguousarray(shard[idx[u]])
                    shard[idx[u]] = 0.0
                    r_u, r_v = _exchange_lists(u, vals, rank ^ (1 << j))
                    shard[idx[r_u]] = r_v
                else:
                    recv = _exchange(torch.from_numpy(np.ascontiguousarray(shard[idx])), rank ^ (1 << j))
                    shard[idx] = recv.numpy()
                qa = int(np.nonzero(perm == gpos)[0][0])
                qb = int(np.nonzero(perm == lpos)[0][0])
                perm[qa], perm[qb] = perm[qb], perm[qa]
            else:  # generator `gen`: its strings, physical masks, global Z as a sign
                for t in range(off[gen], off[gen + 1]):
                    xp, zp = _permute(int(x[t]), perm), _permute(int(z[t]), perm)
                    assert xp >> l == 0, "flip mask must be local after the swaps"
                    sg = -1.0 if bin((rank << l) & zp).count("1") % 2 else 1.0
                    shard = ffo.apply_pauli_rotation(l, shard, xp, zp & mask, sg * theta[gen] * c[t].imag)
        assert np.array_equal(perm, fp)
        # expectation: one whole-shard exchange per distinct out-of-shard flip pattern
        hx, hz, hc = P.ham_arrays()
        xs = np.array([_permute(int(v), perm) for v in hx])
        zs = np.array([_permute(int(v), perm) for v in hz])
        e_local = 0.0 + 0.0j
        kl = np.arange(1 << l)
        kfull = (rank << l) | kl
        for h in sorted(set((xs >> l).tolist())):
            other = shard if h == 0 else _exchange(torch.from_numpy(shard), rank ^ h).numpy()
            for xp, zp, cc in zip(xs, zs, hc):
                if (xp >> l) != h:
                    continue
                ny = bin(xp & zp).count("1")
                par = np.array([bin(v).count("1") & 1 for v in ((kfull ^ xp) & zp)])
                e_local += cc * (1j ** ny) * np.sum(np.conj(shard) * (1 - 2 * par) * other[kl ^ (xp & mask)])
        e = torch.tensor([e_local.real, e_local.imag], dtype=torch.float64)
        dist.all_reduce(e)
        parts = [None] * world
        dist.all_gather_object(parts, shard)
        q.put((rank, e.numpy().tolist(), parts if rank == 0 else None, perm.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,sparse", [(2, False), (4, False), (2, True), (4, True)])
def test_sharded_protocol_across_processes(world, sparse):
    from oracle import ffo

    n, ne, seed = 10, 4, problems.ham_seed(7)
    P = problems.make_problem(n // 2, ne, seed)
    x, z, c = P.ham_arrays()
    H = ffo.PauliSum.from_terms(n, x, z, c)
    kind, idx = ffo.build_generators(n, ne)
    e_ref, _, psi_ref = ffo.energy_trotter(n, ne, kind, idx, np.array(P.plan.order, np.int32), P.thetas[0], H,
                                           want_state=True)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, n, ne, seed, sparse)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = world.bit_length() - 1
    l = n - g
    perm = np.array(res[0][3])
    inv = np.argsort(perm)
    psi = np.zeros(1 << n, complex)
    for r, shard in enumerate(res[0][2]):
        for k in range(1 << l):
            phys = (r << l) | k
            logical = sum(1 << int(inv[pq]) for pq in range(n) if (phys >> pq) & 1)
            psi[logical] = shard[k]
    assert np.abs(psi - psi_ref).max() <= 1e-12
    for _, (er, ei), _, _ in res:
        assert abs(er - e_ref) <= 1e-10 and abs(ei) <= 1e-10
