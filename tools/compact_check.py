"""Compact real sector path (ffq_compact.inl) against the dense support-tracked
path (FFQ_COMPACT=0) on the same inputs, and config-5 timings.
Usage: python tools/compact_check.py [check|time]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_17993_b200 import capi, problems  # noqa: E402


def energy(P, compact, reps=1):
    os.environ["FFQ_COMPACT"] = "1" if compact else "0"
    os.environ.setdefault("FFQ_COMPACT_MIN", "20")
    ctx = capi.Context(0)
    plan = capi.Plan(ctx, P.n_qubits, *P.plan_arrays())
    ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
    s = torch.cuda.ExternalStream(ctx.stream_ptr())
    out = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        e = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())
        b.record(s)
        b.synchronize()
        out.append((e.tolist(), a.elapsed_time(b)))
    n0 = ctx.launches()
    del plan, ham, ctx
    return out


mode = sys.argv[1] if len(sys.argv) > 1 else "check"
if mode == "check":
    cases = [("config5 recipe, 20 q", problems.config5_problem(n_doubles=400, n_terms=300, n_qubits=20, n_elec=10)),
             ("molecular UCCSD, 20 q, 10 e", problems.make_problem(10, 10, problems.ham_seed(9, 1), batch=2)),
             ("molecular UCCSD, 20 q, 8 e", problems.make_problem(10, 8, problems.ham_seed(9, 2), batch=1))]
    for name, P in cases:
        t0 = time.time()
        ec = energy(P, True)[-1]
        ed = energy(P, False)[-1]
        d = max(abs(x - y) for x, y in zip(ec[0], ed[0]))
        print(json.dumps({"case": name, "compact": ec[0], "dense_support": ed[0], "max_abs_diff": d,
                          "ms_compact": ec[1], "ms_dense": ed[1], "wall_s": time.time() - t0}), flush=True)
else:
    for nq in (28, 32):
        P = problems.config5_problem(n_qubits=nq, n_elec=nq // 2)
        r = energy(P, True, reps=3)
        print(json.dumps({"config5_qubits": nq, "energy": r[-1][0], "ms": [x[1] for x in r]}), flush=True)
