"""Device time of the two phases of an 18-qubit energy evaluation (generator
passes vs expectation) through the state-level C-ABI, CUDA events on the
context stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_17993_b200 import capi, problems  # noqa: E402

B = int(os.environ.get("PT_BATCH", "16"))
cfg = int(os.environ.get("PT_CONFIG", "3"))
P = problems.config_problem(cfg, batch=B)
for tb in [int(v) for v in os.environ.get("PT_TILE", "0,12").split(",")]:
    os.environ["FFQ_TILE_BITS"] = str(tb)
    ctx = capi.Context(0)
    plan = capi.Plan(ctx, P.n_qubits, *P.plan_arrays())
    ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
    st = capi.State(ctx, P.n_qubits, B)
    s = torch.cuda.ExternalStream(ctx.stream_ptr())
    th = P.plan_thetas()

    def ev(fn, reps=3):
        fn()
        ctx.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            fn()
        b.record(s)
        b.synchronize()
        return a.elapsed_time(b) / reps

    st.set_basis(P.hf)
    t_plan = ev(lambda: st.apply_plan(plan, th))
    t_exp = ev(lambda: st.expectation(ham))
    print(f"tile_bits={tb} batch={B}: plan {t_plan:.3f} ms ({1e3 * t_plan / B:.1f} us/eval), "
          f"expectation {t_exp:.3f} ms ({1e3 * t_exp / B:.1f} us/eval)", flush=True)
    del st, plan, ham, ctx
