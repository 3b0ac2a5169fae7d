"""HBM roofline of the dense grouped-expectation pass (k_expect_items) and the
dense fused-generator pass (k_fused_gen) on a state of 4 GiB (28 qubits, >> L2):
SPEC.md:419-427's contract at a size where only HBM can feed the pass. The state
is made dense with one X rotation per qubit. FFQ_SUPPORT=0 selects the dense
kernels. Usage: dense_passes.py [n_qubits] [n_terms] [n_generators]"""
import json
import os
import sys

import numpy as np

os.environ["FFQ_SUPPORT"] = "0"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_17993_b200 import capi, problems  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
K = int(sys.argv[2]) if len(sys.argv) > 2 else 16
G = int(sys.argv[3]) if len(sys.argv) > 3 else 24
peak = 6546.6
try:
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
except Exception:
    pass
ctx = capi.Context(0)
stream = torch.cuda.ExternalStream(ctx.stream_ptr())
st = capi.State(ctx, n, 1)
st.set_basis(0)
for q in range(n):
    st.rotate(1 << q, 0, 0.3 + 0.01 * q)
ctx.synchronize()


def timed(fn, reps):
    fn()
    ctx.synchronize()
    ms = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    return float(np.mean(ms))


rng = np.random.default_rng(28)
# K Pauli strings with distinct non-zero flip masks: K x-groups, each one pass of 16 B per amplitude
hx = rng.choice(np.arange(1, 1 << 20, dtype=np.uint64), size=K, replace=False) << np.uint64(n - 20)
hx |= rng.integers(0, 1 << (n - 20), size=K, dtype=np.uint64)
hz = rng.integers(0, 1 << n, size=K, dtype=np.uint64)
ny = np.array([bin(int(a & b)).count("1") for a, b in zip(hx, hz)])
hz = np.where(ny % 2 == 1, hz ^ (hx & (~hx + np.uint64(1))), hz)  # even Y count: Hermitian with real c
ham = capi.Hamiltonian(ctx, n, hx, hz, rng.normal(size=K))
ms_e = timed(lambda: st.expectation(ham), 5)
bytes_e = K * 16 * (1 << n)
print(json.dumps({"pass": "grouped expectation (k_expect_items)", "n_qubits": n, "x_groups": K, "ms": ms_e,
                  "algorithmic_bytes": bytes_e, "achieved_gbs": bytes_e / ms_e / 1e6,
                  "frac_of_measured_hbm_peak": bytes_e / ms_e / 1e6 / peak}), flush=True)

# G fused UCCSD doubles at n qubits, each touching 2^(n-3) amplitudes (r + w): (a) flip
# masks on qubits >= 3 (runs of >= 8 amplitudes = whole 128-byte lines), (b) flip masks
# holding qubits 0 and 1 (one live amplitude per 64-byte DRAM atom of the natural-order
# layout: 4x the algorithmic bytes must move)
P = problems.config5_problem(n_doubles=100000, n_terms=4, n_qubits=n, n_elec=n // 2)
off, x, z, c = P.plan_arrays()
doubles = [g for g in range(len(off) - 1) if off[g + 1] - off[g] == 8]
for label, pick in (("flip masks on qubits >= 3", lambda m: (m & 7) == 0),
                    ("flip masks holding qubits 0 and 1", lambda m: (m & 3) == 3)):
    dbl = [g for g in doubles if pick(int(x[off[g]]))][:G]
    o2 = np.array([0] + list(np.cumsum([8] * len(dbl))), np.int64)
    sel = np.concatenate([np.arange(off[g], off[g + 1]) for g in dbl])
    plan = capi.Plan(ctx, n, o2, x[sel], z[sel], c[sel])
    th = rng.uniform(-0.05, 0.05, size=(1, len(dbl)))
    ms_g = timed(lambda: st.apply_plan(plan, th), 5)
    bytes_g = len(dbl) * 32 * (1 << (n - 3))
    print(json.dumps({"pass": "fused generator (k_fused_gen), " + label, "n_qubits": n, "generators": len(dbl),
                      "ms": ms_g, "ms_per_generator": ms_g / len(dbl), "algorithmic_bytes": bytes_g,
                      "achieved_gbs": bytes_g / ms_g / 1e6,
                      "frac_of_measured_hbm_peak": bytes_g / ms_g / 1e6 / peak}), flush=True)
    del plan
