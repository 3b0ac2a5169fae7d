"""A few generic rotation passes on a 28-qubit state (4 GiB >> L2), the
roofline kernel of bench.py, for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_17993_b200 import capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
ctx = capi.Context(0)
st = capi.State(ctx, n, 1)
st.set_basis(0)
for k in range(4):
    st.rotate(0b1011 << 9, 0b111 << 4, 0.1 * (1 - 2 * (k % 2)))
ctx.synchronize()
print("ok", n)
