"""BASELINE.json config 5 on one B200 (0 global qubits): energy evaluations
through the default path (the compact real sector layout from 27 qubits up),
CUDA-event timed. Usage: config5.py [n_qubits] [batch]; batch > 1 adds seeded
theta rows (the compact layout interleaves 4 rows per matrix)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_17993_b200 import capi, problems  # noqa: E402

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 32
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
t0 = time.time()
P = problems.config5_problem(n_qubits=nq, n_elec=nq // 2)
rows = P.thetas
if batch > 1:
    rows = np.concatenate([rows, np.random.default_rng(5).uniform(-0.05, 0.05, size=(batch - 1, P.n_gen))])
th = P.plan_thetas(rows)
ctx = capi.Context(0)
plan = capi.Plan(ctx, nq, *P.plan_arrays())
ham = capi.Hamiltonian(ctx, nq, *P.ham_arrays())
host_s = time.time() - t0
s = torch.cuda.ExternalStream(ctx.stream_ptr())
out = {}
for rep in range(3):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s)
    e = capi.energy_batch(ctx, plan, ham, P.hf, th)
    b.record(s)
    b.synchronize()
    out[f"rep{rep}"] = {"energy": float(e[0]), "ms": a.elapsed_time(b), "ms_per_eval": a.elapsed_time(b) / batch}
print(json.dumps({"config": 5, "n_qubits": nq, "batch": batch, "generators": P.n_gen, "terms": len(P.H),
                  "host_build_s": host_s, "compact_il": os.environ.get("FFQ_COMPACT_IL", "4"),
                  "path": ("compact real sector layout (ffq_compact.inl), 1 GPU" if nq >= 27 else
                           "support-tracked graph, 1 GPU, 0 global qubits"), **out}),
      flush=True)
