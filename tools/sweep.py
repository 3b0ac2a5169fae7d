"""Throughput sweep of the config-3 energy step over runtime knobs
(FFQ_SLAB_MB and any FFQ_* env list), CUDA-event timed on the context stream."""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_17993_b200 import capi, problems  # noqa: E402

B = int(os.environ.get("SWEEP_BATCH", "256"))
P = problems.config_problem(int(os.environ.get("SWEEP_CONFIG", "3")), batch=max(1, min(B, 64)))
if B > P.thetas.shape[0]:  # tile the seeded theta rows up to the batch size
    P.thetas = np.tile(P.thetas, (-(-B // P.thetas.shape[0]), 1))[:B]
th = torch.from_numpy(P.plan_thetas()).cuda()
e = torch.zeros(B, dtype=torch.float64, device="cuda")
ref = None
slabs = [int(v) for v in os.environ.get("SWEEP_SLAB", "16,64,256,1024").split(",")]
tiles = [int(v) for v in os.environ.get("SWEEP_TILE", "12").split(",")]
envs = [e for e in os.environ.get("SWEEP_ENV", "").split(";")]
base_env = dict(os.environ)
for slab, tb, env in itertools.product(slabs, tiles, envs):
    os.environ.clear()
    os.environ.update(base_env)
    os.environ["FFQ_SLAB_MB"] = str(slab)
    pass  # (FFQ_TILE_BITS: removed with the tiled expectation)
    for kv in filter(None, env.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    ctx = capi.Context(0)
    plan = capi.Plan(ctx, P.n_qubits, *P.plan_arrays())
    ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
    st = torch.cuda.ExternalStream(ctx.stream_ptr())
    f = lambda: capi.energy_batch_device(ctx, plan, ham, P.hf, B, th.data_ptr(), e.data_ptr())  # noqa: E731
    f(); f()
    ctx.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(3):
        f()
    b.record(st)
    b.synchronize()
    ms = a.elapsed_time(b) / 3
    out = e.cpu().numpy()
    if ref is None:
        ref = out.copy()
    print(json.dumps({"slab_mb": slab, "tile_bits": tb, "env": env, "ms_per_batch": ms, "evals_per_s": B / ms * 1e3,
                      "max_dev_vs_first": float(np.abs(out - ref).max())}), flush=True)
    del plan, ham, ctx
