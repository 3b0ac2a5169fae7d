"""Per-phase cycles (FFQ_PHASE_CLOCKS) of the config-3 support-closure program
for one launch of B evaluations, plus CUDA-event throughput of the same launch."""
import os
import sys

os.environ.setdefault("FFQ_PHASE_CLOCKS", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_17993_b200 import capi, problems  # noqa: E402

B = int(os.environ.get("PT_BATCH", "148"))
P = problems.config_problem(int(os.environ.get("PT_CONFIG", "3")), batch=min(B, 64))
th = np.tile(P.plan_thetas(), (-(-B // P.thetas.shape[0]), 1))[:B]
ctx = capi.Context(0)
plan = capi.Plan(ctx, P.n_qubits, *P.plan_arrays())
ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
for _ in range(2):
    e = capi.energy_batch(ctx, plan, ham, P.hf, th)
print("e0", e[0], flush=True)
