"""One chunk of the config-3 energy step, for ncu launch lists / full captures.
Usage: python tools/profile_step.py [--batch 16] [--reps 2] [--config 3]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2402_17993_b200 import capi, problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--config", type=int, default=3)
a = ap.parse_args()
P = problems.config_problem(a.config, batch=a.batch)
ctx = capi.Context(0)
plan = capi.Plan(ctx, P.n_qubits, *P.plan_arrays())
ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
for r in range(a.reps):
    e = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())
print("launches", ctx.launches(), "e0", e[0])
