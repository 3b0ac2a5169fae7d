"""Small runs of every execution path for compute-sanitizer (memcheck/racecheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2402_17993_b200 import capi, problems  # noqa: E402

for env in ({}, {"FFQ_SMEM_MAX_QUBITS": "0"}, {"FFQ_SMEM_MAX_QUBITS": "0", "FFQ_SUPPORT": "0"},
            ):
    os.environ.update(env)
    ctx = capi.Context(0)
    P = problems.make_problem(7, 6, problems.ham_seed(9), batch=3)
    plan = capi.Plan(ctx, P.n_qubits, *P.plan_arrays())
    ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
    e = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())
    st = capi.State(ctx, P.n_qubits, 2)
    st.set_basis(P.hf)
    st.apply_plan(plan, np.repeat(P.plan_thetas()[:1], 2, axis=0))
    st.rotate(0b1011, 0b110, 0.3)
    st.expectation(ham)
    sh = capi.ShardedState(ctx, P.n_qubits, 2)
    sh.energy(plan, ham, P.hf, P.plan_thetas()[0])
    print(env, e.tolist())
    for k in env:
        del os.environ[k]
print("sanitize smoke ok")
