"""B = 1 latency of the config-3 energy with L2 flushed before every timed call
(the bench's secondary.config3_latency_and_b64.b1_ms), per FFQ_* setting given
in LAT_ENV (';'-separated, one child process each). LAT_BATCH=b1,b2,...: the
same for small batches (ms per call)."""
import json
import os
import statistics
import subprocess
import sys

ENVS = os.environ.get("LAT_ENV", "FFQ_WARM=1;FFQ_WARM=0").split(";")
if len(ENVS) > 1:
    for env in ENVS:
        r = subprocess.run([sys.executable, __file__], env={**os.environ, "LAT_ENV": env}, capture_output=True, text=True)
        sys.stdout.write(r.stdout if r.returncode == 0 else json.dumps({"env": env, "error": r.stderr[-400:]}) + "\n")
    sys.exit(0)
for kv in filter(None, ENVS[0].split(",")):
    k, v = kv.split("=")
    os.environ[k] = v
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_17993_b200 import capi, problems  # noqa: E402

BATCHES = [int(b) for b in os.environ.get("LAT_BATCH", "1").split(",")]
P = problems.config_problem(3, batch=max(BATCHES))
th = torch.from_numpy(P.plan_thetas()).cuda()
e = torch.zeros(max(BATCHES), dtype=torch.float64, device="cuda")
ctx = capi.Context(0)
plan = capi.Plan(ctx, P.n_qubits, *P.plan_arrays())
ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
s = torch.cuda.ExternalStream(ctx.stream_ptr())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {"env": ENVS[0]}
for B in BATCHES:
    f = lambda: capi.energy_batch_device(ctx, plan, ham, P.hf, B, th.data_ptr(), e.data_ptr())  # noqa: E731
    for _ in range(3):
        f()
    ctx.synchronize()
    ms = []
    with torch.cuda.stream(s):
        for _ in range(20):
            flush.fill_(1)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            f()
            b.record(s)
            b.synchronize()
            ms.append(a.elapsed_time(b))
    out["b1_cold_ms" if B == 1 else "b%d_cold_ms" % B] = statistics.median(ms)
out["energy"] = float(e[0].item())
print(json.dumps(out), flush=True)
