"""BASELINE.json config 5 on one B200 (0 global qubits; a 64 GiB state fits):
one energy evaluation through the support-tracked graph path, CUDA-event timed,
plus the sharded path (group emulation) at a reduced qubit count."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_17993_b200 import capi, problems  # noqa: E402

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 32
t0 = time.time()
P = problems.config5_problem(n_qubits=nq, n_elec=nq // 2)
ctx = capi.Context(0)
plan = capi.Plan(ctx, nq, *P.plan_arrays())
ham = capi.Hamiltonian(ctx, nq, *P.ham_arrays())
host_s = time.time() - t0
s = torch.cuda.ExternalStream(ctx.stream_ptr())
out = {}
for rep in range(2):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s)
    e = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())[0]
    b.record(s)
    b.synchronize()
    out[f"rep{rep}"] = {"energy": e, "ms": a.elapsed_time(b)}
print(json.dumps({"config": 5, "n_qubits": nq, "generators": P.n_gen, "terms": len(P.H),
                  "host_build_s": host_s, "path": ("compact real sector layout (ffq_compact.inl), 1 GPU" if nq >= 27 else
                          "support-tracked graph, 1 GPU, 0 global qubits"), **out}),
      flush=True)
