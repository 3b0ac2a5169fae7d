"""a15 at full size: BASELINE.json config 5 (32 qubits, 16
electrons, 128 singles + the first 2000 doubles, 5000 random Pauli terms)
through the sharded state in group mode on ONE B200: 2^3 shards of 2^29
amplitudes (8 GiB each, 64 GiB total) split on 3 global qubits, every global
touch a pairwise half-shard swap with the same k_swap_pack/unpack kernels as
the NCCL transport (a device copy as the wire), the expectation one partner
exchange per out-of-shard flip pattern. Its energy is compared with the
compact real sector layout (the default 32-qubit path). One JSON line.

Usage: python tools/shard32.py [n_qubits] [n_global]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_17993_b200 import capi, problems  # noqa: E402

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 32
g = int(sys.argv[2]) if len(sys.argv) > 2 else 3
P = problems.config5_problem(n_qubits=nq, n_elec=nq // 2)
ctx = capi.Context(0)
plan = capi.Plan(ctx, nq, *P.plan_arrays())
ham = capi.Hamiltonian(ctx, nq, *P.ham_arrays())
th = P.plan_thetas()[0]
stream = torch.cuda.ExternalStream(ctx.stream_ptr())

t = time.time()
e_compact = float(capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())[0])
t_compact = time.time() - t

off, x, z, c = P.plan_arrays()
_, _, sw, _ = capi.shard_schedule(nq, g, off, x, z, c)
sh = capi.ShardedState(ctx, nq, g)
runs = []
for rep in range(2):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    e = sh.energy(plan, ham, P.hf, th)
    b.record(stream)
    b.synchronize()
    runs.append({"energy": e, "ms": a.elapsed_time(b)})
swaps, perm = sh.info()
free, total = torch.cuda.mem_get_info()
print(json.dumps({
    "config": 5, "n_qubits": nq, "global_qubits": g, "shards": 1 << g, "shard_gib": (16 << (nq - g)) / 2 ** 30,
    "generators": P.n_gen, "terms": len(P.H), "swaps_per_eval": swaps, "scheduled_swaps": int(sw),
    "sharded": runs, "bitwise_repeatable": runs[0]["energy"] == runs[1]["energy"],
    "compact_energy": e_compact, "compact_first_call_s": t_compact,
    "abs_diff_vs_compact": abs(runs[0]["energy"] - e_compact),
    "device_mem_used_gib": (total - free) / 2 ** 30,
    "path": "group mode: every shard on this device; the NCCL transport runs the same kernels with "
            "ncclSend/ncclRecv as the wire"}), flush=True)
