"""One rank of the sharded-state path over NCCL: BASELINE
config 5's recipe at n qubits split on g = log2(world) global qubits, one
process per GPU, half-shard swaps by ncclSend/ncclRecv. bench.py starts one of
these per rank (a child process, so a transport failure cannot take the bench
line with it) and passes the NCCL unique id made by rank 0.

Usage: shard_nccl_leg.py n_qubits n_global rank nccl_id_hex|self device [reps]
Prints one JSON line: energy, ms per evaluation (CUDA events on the context
stream, after one warm-up evaluation), swaps per evaluation."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_17993_b200 import capi, problems  # noqa: E402

nq, g, rank = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
nccl_id = capi.nccl_unique_id() if sys.argv[4] == "self" else bytes.fromhex(sys.argv[4])  # "self": world 1
dev = int(sys.argv[5])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 2
P = problems.config5_problem(n_qubits=nq, n_elec=nq // 2)
ctx = capi.Context(dev)
plan = capi.Plan(ctx, nq, *P.plan_arrays())
ham = capi.Hamiltonian(ctx, nq, *P.ham_arrays())
th = P.plan_thetas()[0]
torch.cuda.set_device(dev)
stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=torch.device("cuda", dev))
sh = capi.ShardedState(ctx, nq, g, rank=rank, nccl_id=nccl_id)
e = sh.energy(plan, ham, P.hf, th)  # warm-up: schedules, physical Hamiltonian, NCCL channels
ms = []
for _ in range(reps):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    e2 = sh.energy(plan, ham, P.hf, th)
    b.record(stream)
    b.synchronize()
    ms.append(a.elapsed_time(b))
swaps, _ = sh.info()
print(json.dumps({"rank": rank, "n_qubits": nq, "global_qubits": g, "energy": e2, "repeatable": e == e2,
                  "ms_per_eval": sum(ms) / len(ms), "swaps_per_eval": swaps,
                  "shard_gib": (16 << (nq - g)) / 2 ** 30}), flush=True)
