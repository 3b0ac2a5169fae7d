"""Production-size runs of the barrier-pipelined shared-memory kernels for
compute-sanitizer racecheck / synccheck (one kernel family per argv[1]):

  real     k_sector_eval_real at config 3 (18 qubits, 1024 threads, alpha-beta
           cliques + anchored blocks + generic rows), batch 2 (split CTAs)
  complex  k_sector_eval<2,768> at config 3 (2-CTA cluster, DSMEM peer copies)
  runs     k_rotation_run at 20 qubits: low-12 TMA tiles and gathered tiles
  smoke    every other execution path at 14 qubits (tools/sanitize_smoke.py)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2402_17993_b200 import capi, problems  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "real"
if which in ("real", "complex"):
    if which == "complex":
        os.environ["FFQ_SECTOR_REAL"] = "0"
    ctx = capi.Context(0)
    P = problems.config_problem(3, batch=2)
    plan = capi.Plan(ctx, P.n_qubits, *P.plan_arrays())
    ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
    info = capi.sector_info(ctx, plan, ham, P.hf)
    e = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())
    print(which, "real" if info["real_amplitudes"] else "complex", info["ctas_per_eval"], e.tolist())
elif which == "runs":
    ctx = capi.Context(0)
    n = 20
    rng = np.random.default_rng(3)
    st = capi.State(ctx, n, 1)
    psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    st.upload(psi / np.linalg.norm(psi))
    x_low = rng.integers(1, 1 << 12, size=8, dtype=np.uint64)
    x_gat = np.array([int(v) | (1 << 19) | (1 << 15) for v in rng.integers(0, 32, size=8)], np.uint64)
    for x in (x_low, x_gat):
        z = rng.integers(0, 1 << n, size=len(x), dtype=np.uint64)
        st.rotate_many(x, z, rng.uniform(-1, 1, size=len(x)))
    print("runs", float(np.linalg.norm(st.download()[0])))
print("sanitize", which, "ok")
