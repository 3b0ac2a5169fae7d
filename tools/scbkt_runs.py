"""SCBKT config-3 energies (16 qubits, per-string rotation ops) with and
without fused low-qubit runs (FFQ_ROT_TILE): evals/s and launches per call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_17993_b200 import capi, problems  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
R = problems.config_problem(3, batch=B, mapping="scbkt")
for tile in ("12", "0"):
    os.environ["FFQ_ROT_TILE"] = tile
    c = capi.Context(0)
    plan = capi.Plan(c, R.n_qubits, *R.plan_arrays())
    ham = capi.Hamiltonian(c, R.n_qubits, *R.ham_arrays())
    th = R.plan_thetas()
    e = capi.energy_batch(c, plan, ham, R.hf, th)
    l0 = c.launches()
    t = time.perf_counter()
    for _ in range(3):
        e = capi.energy_batch(c, plan, ham, R.hf, th)
    dt = (time.perf_counter() - t) / 3
    print(f"FFQ_ROT_TILE={tile}: {B / dt:.0f} evals/s ({dt * 1e3:.2f} ms per {B}-row call), "
          f"{(c.launches() - l0) // 3} launches per call, e[0]={e[0]:.12f}", flush=True)
    del plan, ham
    c.close()
