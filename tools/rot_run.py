"""Fused low-qubit rotation runs (k_rotation_run) on a 28-qubit state: time per
run of R rotations against R single passes (k_pauli_rotation), for ncu captures
and quick timing. Usage: rot_run.py [n] [R]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_17993_b200 import capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
R = int(sys.argv[2]) if len(sys.argv) > 2 else 16
ctx = capi.Context(0)
st = capi.State(ctx, n, 1)
st.set_basis(0)
rr = np.random.default_rng(11)
x = rr.integers(1, 1 << 12, size=R, dtype=np.uint64)
if os.environ.get("ROT_HIGH"):  # flip masks on qubits 0-4 and n-7..n-1: gather tiles (not the low 12)
    x = np.array([(int(v) & 31) | ((int(v) >> 5) << (n - 7)) for v in x], np.uint64)
z = rr.integers(0, 1 << n, size=R, dtype=np.uint64)
th = rr.uniform(-1, 1, size=R)
reps = int(os.environ.get("ROT_REPS", "6"))
for _ in range(2):
    st.rotate_many(x, z, th)
ctx.synchronize()
t = time.perf_counter()
for _ in range(reps):
    st.rotate_many(x, z, th)
ctx.synchronize()
dt = (time.perf_counter() - t) / reps
t = time.perf_counter()
for r in range(R):
    st.rotate(int(x[r]), int(z[r]), float(th[r]))
ctx.synchronize()
du = time.perf_counter() - t
print(f"n={n} R={R}{' high-qubit masks' if os.environ.get('ROT_HIGH') else ''}: fused {dt*1e3:.3f} ms/run ({32*(1<<n)/dt/1e9:.0f} GB/s), unfused {du*1e3:.3f} ms "
      f"({du/dt:.2f}x)")
