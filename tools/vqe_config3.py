"""BASELINE.json config 3 VQE loop on one B200: BFGS driven by batched exact
gradients (four-term rule, 4 x 560 shifted energies per gradient in one call)
through the C++ optimizer and the C-ABI energy batch. Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2402_17993_b200 as ff  # noqa: E402
from paper_2402_17993_b200 import capi, problems  # noqa: E402

max_evals = int(sys.argv[1]) if len(sys.argv) > 1 else 60000
P = problems.config_problem(3)
ctx = capi.Context(0)
plan = capi.Plan(ctx, P.n_qubits, *P.plan_arrays())
ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
order = np.asarray(P.plan.order)
trace = []


def batch_energy(X, B):
    X = np.asarray(X).reshape(B, P.n_gen)
    e = capi.energy_batch(ctx, plan, ham, P.hf, np.ascontiguousarray(X[:, order]))
    if B == 1:
        trace.append(float(e[0]))
    return list(e)


opts = ff.OptimizerOptions()
opts.ftol = 1e-8
opts.max_evals = max_evals
e0 = batch_energy(P.thetas[0], 1)[0]
t = time.time()
r = ff.bfgs_minimize(batch_energy, list(P.thetas[0]), opts)
dt = time.time() - t
zero = capi.energy_batch(ctx, plan, ham, P.hf, np.zeros((1, P.n_gen)))[0]
print(json.dumps({"config": 3, "optimizer": "BFGS + exact 4-term gradients (batched)", "e_initial": e0,
                  "e_hf": zero, "e_final": r.energy, "converged": r.converged, "iterations": r.n_iterations,
                  "energy_evaluations": r.n_evals, "wall_s": dt, "evals_per_s_wall": r.n_evals / dt,
                  "energy_trace_first": trace[:5], "energy_trace_last": trace[-5:]}), flush=True)
