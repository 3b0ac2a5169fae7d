import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2402_17993_b200 import capi
from oracle import ffo
n = 14
rng = np.random.default_rng(0)
psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
psi /= np.linalg.norm(psi)
cases = {"diag Z3": ([0], [8]), "X1X2": ([6], [0]), "X13": ([1 << 13], [0]), "X0X13": ([1 | 1 << 13], [0]),
         "Y5Y12": ([(1 << 5) | (1 << 12)], [(1 << 5) | (1 << 12)]), "X12X13Z0": ([3 << 12], [1]),
         "X2X12Z13": ([(1 << 2) | (1 << 12)], [1 << 13])}
for tb in (0, 12):
    os.environ["FFQ_TILE_BITS"] = str(tb)
    ctx = capi.Context(0)
    st = capi.State(ctx, n, 1)
    st.upload(psi)
    for name, (x, z) in cases.items():
        H = capi.Hamiltonian(ctx, n, x, z, [0.7])
        got = st.expectation(H)[0]
        ref = ffo.expectation(n, psi, ffo.PauliSum.from_terms(n, x, z, [0.7]))
        print(tb, name, "gpu", got.real, "oracle", ref.real, "diff", abs(got.real - ref.real))
