"""Generate tests/golden/energies.json: golden energies (and one full state)
for BASELINE.json configs 1-3 on their seeded synthetic inputs.

The reference has no implementation or golden vectors for this path (SURVEY.md
8c), so the values come from the C oracle (oracle/ffo_oracle.c, the SPEC.md
restatement), cross-checked here against three independent computations: a
dense-matrix <psi|H|psi> for config 1; for EVERY row of configs 1-3, the
oracle's JW-free evaluator (ffo.energy_fermionic: Givens rotations on
determinants and <H> from the second-quantised h, g; no Pauli strings); and
scipy sparse matrix exponentials exp(theta_g A_g) of every generator's JW image
with <H> from the Pauli index action (tests/sparse_ref.py: no closed-form
rotation, no fused patterns; every row of configs 1-2, the first row of config
3). All must agree to <= 1e-12 Hartree. The fixtures pin the oracle (tests/test_golden.py)
and the CUDA path (tests/test_gpu_parity.py) against drift. Floats are stored
as hex strings (exact round trip).

Usage: python tools/make_golden.py   (CPU only; ~3 min, of which ~95 s for the config-3 sparse-matrix row)
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import ffo  # noqa: E402
from oracle import workload as ow  # noqa: E402
from paper_2402_17993_b200 import problems  # noqa: E402

import dense  # noqa: E402
import sparse_ref  # noqa: E402

ROWS = {1: 8, 2: 4, 3: 2}


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    out = {"generator": "tools/make_golden.py",
           "source": "C oracle (oracle/ffo_oracle.c); cross-checked against dense matrices (config 1), the JW-free "
                     "determinant evaluator (every row) and scipy sparse matrix exponentials (tests/sparse_ref.py)",
           "configs": {}}
    for cfg, nrows in ROWS.items():
        P = problems.config_problem(cfg, batch=nrows)
        x, z, c = P.ham_arrays()
        H = ffo.PauliSum.from_terms(P.n_qubits, x, z, c)
        kind, idx = ffo.build_generators(P.n_qubits, P.n_elec)
        order = np.array(P.plan.order, np.int32)
        rows = []
        OP = ow.config_problem(cfg, batch=nrows)  # integrals from the oracle alone
        assert np.array_equal(OP.thetas, P.thetas) and np.array_equal(OP.order, order)
        ferm_dev = 0.0
        expm_dev = 0.0
        expm_rows = 0
        for b in range(nrows):
            want_state = cfg == 1 and b == 0
            r = ffo.energy_trotter(P.n_qubits, P.n_elec, kind, idx, order, P.thetas[b], H, want_state=want_state)
            e, im = r[0], r[1]
            assert abs(im) <= 1e-12
            ef = ffo.energy_fermionic(OP.h, OP.g, OP.n_elec, OP.kind, OP.idx, OP.order, P.thetas[b])
            assert abs(ef - e) <= 1e-12, (cfg, b, ef, e)
            ferm_dev = max(ferm_dev, abs(ef - e))
            # third evaluator: scipy sparse matrix exponentials exp(theta_g A_g) and the Pauli index action
            # (every row at configs 1-2; the first row at config 3: ~95 s)
            if cfg < 3 or b == 0:
                es, ps = sparse_ref.energy(P.n_qubits, P.hf, P.plan_arrays(), P.plan_thetas()[b], P.ham_arrays())
                assert abs(es.real - e) <= 1e-12 and abs(es.imag) <= 1e-12, (cfg, b, es, e)
                assert abs(np.linalg.norm(ps) - 1.0) <= 1e-12
                expm_dev = max(expm_dev, abs(es.real - e))
                expm_rows += 1
            row = {"theta_canonical": [float(t).hex() for t in P.thetas[b]], "energy": float(e).hex()}
            if want_state:
                psi = r[2]
                # independent check: <psi|H|psi> with the dense matrix of the Pauli sum
                Hd = dense.psum_dense(P.n_qubits, x, z, c)
                ed = float(np.real(np.vdot(psi, Hd @ psi)))
                assert abs(ed - e) <= 1e-12, (ed, e)
                assert abs(np.linalg.norm(psi) - 1.0) <= 1e-12
                row["state_re"] = [float(v).hex() for v in psi.real]
                row["state_im"] = [float(v).hex() for v in psi.imag]
            rows.append(row)
        out["configs"][str(cfg)] = {
            "n_qubits": P.n_qubits, "n_elec": P.n_elec, "hf": P.hf, "n_gen": P.n_gen, "n_terms": int(len(x)),
            "ham_sha256": digest(x, z, c), "plan_order_sha256": digest(order),
            "jw_free_max_abs_dev": ferm_dev, "sparse_expm_max_abs_dev": expm_dev, "sparse_expm_rows": expm_rows,
            "rows": rows}
        print(f"config {cfg}: {nrows} rows, E0 = {float.fromhex(rows[0]['energy']):.12f}", flush=True)
    path = os.path.join(ROOT, "tests", "golden", "energies.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
