import os, sys
sys.path.insert(0, os.getcwd())
from paper_2402_17993_b200 import capi, problems
nq = int(sys.argv[1])
P = problems.config5_problem(n_qubits=nq, n_elec=nq // 2)
ctx = capi.Context(0)
plan = capi.Plan(ctx, nq, *P.plan_arrays()); ham = capi.Hamiltonian(ctx, nq, *P.ham_arrays())
print(capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas()))
