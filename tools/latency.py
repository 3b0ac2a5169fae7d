"""Single-evaluation latency of the config-3 energy (B = 1) per execution path,
CUDA events on the context stream, mean of 20 calls after warm-up.

LAT_ENV is a ';'-separated list of env settings; each runs in its own child
process because the library reads its FFQ_* knobs once per process."""
import json
import os
import subprocess
import sys

ENVS = os.environ.get("LAT_ENV", "FFQ_SECTOR_CL=2;FFQ_SECTOR_CL=4;FFQ_SECTOR_CL=8;FFQ_SECTOR=0").split(";")

if len(ENVS) > 1:
    for env in ENVS:
        r = subprocess.run([sys.executable, __file__], env={**os.environ, "LAT_ENV": env},
                           capture_output=True, text=True)
        sys.stdout.write(r.stdout if r.returncode == 0 else json.dumps({"env": env, "error": r.stderr[-400:]}) + "\n")
        sys.stdout.flush()
    sys.exit(0)

env = ENVS[0]
for kv in filter(None, env.split(",")):
    k, v = kv.split("=")
    os.environ[k] = v

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_17993_b200 import capi, problems  # noqa: E402

P = problems.config_problem(int(os.environ.get("LAT_CONFIG", "3")))
th = torch.from_numpy(P.plan_thetas()).cuda()
e = torch.zeros(1, dtype=torch.float64, device="cuda")
ctx = capi.Context(0)
plan = capi.Plan(ctx, P.n_qubits, *P.plan_arrays())
ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
s = torch.cuda.ExternalStream(ctx.stream_ptr())
f = lambda: capi.energy_batch_device(ctx, plan, ham, P.hf, 1, th.data_ptr(), e.data_ptr())  # noqa: E731
for _ in range(3):
    f()
ctx.synchronize()
a = torch.cuda.Event(enable_timing=True)
b = torch.cuda.Event(enable_timing=True)
a.record(s)
for _ in range(20):
    f()
b.record(s)
b.synchronize()
print(json.dumps({"env": env, "latency_ms": a.elapsed_time(b) / 20, "energy": float(e.item())}), flush=True)
