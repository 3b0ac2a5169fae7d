"""fragfield command line for the UCCSD hot path.

  python -m paper_2402_17993_b200.cli ham --config 3 --out c3.fcidump
  python -m paper_2402_17993_b200.cli energy --fcidump c3.fcidump --batch 64 [--mapping scbkt]
  python -m paper_2402_17993_b200.cli vqe --config 1 --optimizer bfgs
  python -m paper_2402_17993_b200.cli selftest

Every command prints one JSON RunReport (records per unit: method, HF energy,
correlation energy, total, evaluations, wall time; a provenance block with
hashes of the arguments and inputs). Exit codes: 0 success, 2
numerical non-convergence, 1 usage or input error. The SCF-driven `fmo`/`sc`
subcommands of the reference spec need the integral/SCF chain, which is out of
this repo's scope: Hamiltonians come from FCIDUMP files
or the seeded synthetic configs.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np


def _report(cmd, args, records, inputs=()):
    h = hashlib.sha256(json.dumps(vars(args), sort_keys=True, default=str).encode()).hexdigest()
    prov = {"command": cmd, "config_sha256": h}
    for path in inputs:
        with open(path, "rb") as f:
            prov["input_sha256:" + os.path.basename(path)] = hashlib.sha256(f.read()).hexdigest()
    return {"records": records, "provenance": prov}


def _problem(args, batch=1):
    from . import problems, read_fcidump

    if getattr(args, "fcidump", None):
        h, g, e_const, ne, _ = read_fcidump(args.fcidump)
        return problems.problem_from_integrals(h, g, ne, e_const, seed=args.seed, batch=batch,
                                               theta_hw=args.theta_hw, name=os.path.basename(args.fcidump),
                                               mapping=args.mapping)
    return problems.config_problem(args.config, batch=batch, mapping=args.mapping)


def _device(P):
    from . import capi

    ctx = capi.Context(0)
    return ctx, capi.Plan(ctx, P.n_qubits, *P.plan_arrays()), capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())


def cmd_ham(args):
    from . import problems, write_fcidump

    P = problems.config_problem(args.config)
    write_fcidump(args.out, P.h, P.g, P.n_elec)
    return _report("ham", args, [{"unit": P.name, "norb": P.m, "nelec": P.n_elec, "path": args.out}])


def cmd_energy(args):
    from . import capi

    P = _problem(args, batch=args.batch)
    ctx, plan, ham = _device(P)
    t = time.time()
    e_hf = float(capi.energy_batch(ctx, plan, ham, P.hf, np.zeros((1, P.n_gen)))[0])
    e = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())
    dt = time.time() - t
    recs = [{"unit": P.name, "row": b, "method": f"uccsd-trotter ({P.mapping})", "hf_energy": e_hf,
             "correlation": float(e[b]) - e_hf, "total": float(e[b]), "n_evals": 1} for b in range(len(e))]
    rep = _report("energy", args, recs, [args.fcidump] if args.fcidump else [])
    rep["wall_s"] = dt
    rep["n_qubits"] = P.n_qubits
    return rep


def cmd_vqe(args):
    import paper_2402_17993_b200 as ff
    from . import capi

    P = _problem(args)
    ctx, plan, ham = _device(P)
    order = np.asarray(P.plan.order)

    def batch_energy(X, B):
        X = np.asarray(X).reshape(B, P.n_gen)
        return list(capi.energy_batch(ctx, plan, ham, P.hf, np.ascontiguousarray(X[:, order])))

    opts = ff.OptimizerOptions()
    opts.ftol = args.ftol
    opts.max_evals = args.max_evals
    t = time.time()
    e_hf = batch_energy(np.zeros(P.n_gen), 1)[0]
    if args.optimizer == "bfgs":
        r = ff.bfgs_minimize(batch_energy, list(P.thetas[0]), opts)
    else:
        r = ff.vqe_minimize(lambda x: batch_energy(x, 1)[0], list(P.thetas[0]), args.optimizer, opts)
    rec = {"unit": P.name, "method": f"uccsd-trotter VQE ({args.optimizer}, {P.mapping})", "hf_energy": e_hf,
           "correlation": r.energy - e_hf, "total": r.energy, "n_evals": r.n_evals, "converged": r.converged,
           "wall_s": time.time() - t}
    rep = _report("vqe", args, [rec], [args.fcidump] if args.fcidump else [])
    if not r.converged:
        rep["error"] = "ConvergenceError: optimizer did not reach ftol"
    return rep


GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                      "energies.json")


def cmd_selftest(args):
    """The CUDA path against the committed golden fixtures (tests/golden/energies.json,
    tools/make_golden.py): config-1 energies of every fixture row (<= 1e-10 Ha) and
    the config-1 state after the plan (<= 1e-12 max-abs)."""
    from . import capi, problems

    if not os.path.exists(GOLDEN):
        raise OSError(f"selftest: golden fixtures not found at {GOLDEN}")
    with open(GOLDEN) as f:
        g = json.load(f)["configs"]["1"]
    rows = g["rows"]
    th = np.array([[float.fromhex(t) for t in r["theta_canonical"]] for r in rows])
    P = problems.config_problem(1, batch=len(rows))
    if not np.array_equal(th, P.thetas):
        raise ValueError("selftest: seeded config-1 theta rows differ from the golden fixtures")
    ctx, plan, ham = _device(P)
    e = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())
    de = max(abs(float(e[b]) - float.fromhex(r["energy"])) for b, r in enumerate(rows))
    st = capi.State(ctx, P.n_qubits, 1)
    st.set_basis(P.hf)
    st.apply_plan(plan, P.plan_thetas()[:1])
    psi = st.download()[0]
    ref = np.array([float.fromhex(v) for v in rows[0]["state_re"]]) + 1j * np.array(
        [float.fromhex(v) for v in rows[0]["state_im"]])
    ds = float(np.abs(psi - ref).max())
    ok = de <= 1e-10 and ds <= 1e-12
    rep = _report("selftest", args, [{"unit": "config1", "method": "golden fixtures", "rows": len(rows),
                                      "max_energy_err": de, "max_state_err": ds, "ok": ok}], [GOLDEN])
    if not ok:
        raise ValueError(f"selftest: CUDA path differs from the golden fixtures (energy {de:.3g}, state {ds:.3g})")
    return rep


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="fragfield")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("ham", help="write a synthetic config's Hamiltonian as FCIDUMP")
    p.add_argument("--config", type=int, choices=(1, 2, 3), required=True)
    p.add_argument("--out", required=True)
    for name in ("energy", "vqe"):
        p = sub.add_parser(name)
        src = p.add_mutually_exclusive_group(required=True)
        src.add_argument("--fcidump")
        src.add_argument("--config", type=int, choices=(1, 2, 3))
        p.add_argument("--mapping", choices=("jw", "scbkt"), default="jw")
        p.add_argument("--seed", type=int, default=2402179930)
        p.add_argument("--theta-hw", type=float, default=0.1)
        if name == "energy":
            p.add_argument("--batch", type=int, default=1)
        else:
            p.add_argument("--optimizer", choices=("powell", "neldermead", "bfgs"), default="bfgs")
            p.add_argument("--ftol", type=float, default=1e-8)
            p.add_argument("--max-evals", type=int, default=200000)
    sub.add_parser("selftest")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 1 if e.code else 0
    try:
        rep = {"ham": cmd_ham, "energy": cmd_energy, "vqe": cmd_vqe, "selftest": cmd_selftest}[args.cmd](args)
    except (ValueError, OSError) as e:  # ContractViolation / ParseError are ValueErrors
        print(json.dumps({"error": f"{type(e).__name__}: {e}"}))
        return 1
    except RuntimeError as e:
        print(json.dumps({"error": f"{type(e).__name__}: {e}"}))
        return 2 if "Convergence" in type(e).__name__ else 1
    print(json.dumps(rep))
    return 2 if "error" in rep else 0


if __name__ == "__main__":
    sys.exit(main())
