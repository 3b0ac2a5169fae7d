"""BASELINE.json config 3 VQE loop on one B200.

  BFGS   exact gradients (four-term rule: 4 x 560 shifted energies per gradient,
         one batched call each): fragfield::vqe_bfgs, the device objective in C++
  Powell the paper's derivative-free optimizer on the B = 1 path (one energy per
         call), from the same start

Both to ftol 1e-8 (|dE| of an accepted step). Reports E_final, evaluations,
wall time including the first call's program compile, and the variational
bound against E_CASCI (lanczos_ground). One JSON line
per optimizer.

Usage: python tools/vqe_config3.py [bfgs_max_evals] [powell_max_evals]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2402_17993_b200 as ff  # noqa: E402
from paper_2402_17993_b200 import capi, problems  # noqa: E402

bfgs_max = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
powell_max = int(sys.argv[2]) if len(sys.argv) > 2 else 400_000
t_all = time.time()
P = problems.config_problem(3)
dev = ff.Device(0)
H_dev = ff.DeviceHamiltonian(dev, P.H)
P_dev = ff.DevicePlan(dev, P.plan)
ctx = capi.Context(0)  # CAS-CI reference (lanczos_ground) through the C-ABI binding
ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())

t0 = time.time()
e0 = ff.energy_trotter(dev, list(P.thetas[0]), P_dev, H_dev, P.hf)  # compiles the sector program
t_compile = time.time() - t0
e_hf = ff.energy_trotter(dev, [0.0] * P.n_gen, P_dev, H_dev, P.hf)
gs = capi.lanczos_ground(ctx, ham, P.hf)
e_cas = gs["energy"] if isinstance(gs, dict) else gs[0]

for name, max_evals in (("bfgs", bfgs_max), ("powell", powell_max)):
    opts = ff.OptimizerOptions()
    opts.ftol = 1e-8
    opts.max_evals = max_evals
    t = time.time()
    # the C++ drivers: the objective is the device batch call, no Python in the loop
    if name == "bfgs":
        r = ff.vqe_bfgs(dev, P_dev, H_dev, P.hf, list(P.thetas[0]), opts)
    else:
        r = ff.vqe_device(dev, P_dev, H_dev, P.hf, list(P.thetas[0]), "powell", opts)
    dt = time.time() - t
    print(json.dumps({
        "config": 3, "optimizer": name, "detail": ("BFGS + exact 4-term gradients (4 x 560 rows per batched call), "
                                                   "C++ driver (vqe_bfgs)"
                                                   if name == "bfgs" else "Powell on the B = 1 path, C++ driver (vqe_device)"),
        "e_initial": e0, "e_hf": e_hf, "e_casci": e_cas, "e_final": r.energy,
        "above_casci": r.energy - e_cas, "variational_bound_ok": bool(r.energy >= e_cas - 1e-10),
        "converged": bool(r.converged), "iterations": r.n_iterations, "energy_evaluations": r.n_evals,
        "wall_s": dt, "first_call_compile_s": t_compile, "wall_s_incl_compile": dt + t_compile,
        "evals_per_s_wall": r.n_evals / dt}), flush=True)
print(json.dumps({"total_wall_s": time.time() - t_all}), flush=True)
