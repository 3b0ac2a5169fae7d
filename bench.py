#!/usr/bin/env python3
"""Benchmark: UCCSD energy evals/sec at 18 qubits (complex128) + rotation-pass HBM GB/s.

Step = one VQE gradient evaluation of BASELINE.json config 3 (18 qubits, 10
electrons, 560 generators): the parameter-shift set {theta, theta +- pi/2 e_k}
= 1121 energy evaluations in one batched call through the C-ABI.

  value     device-resident theta/energies (ffq_energy_batch_device), CUDA events
  e2e       host theta in, host energies out (ffq_energy_batch), H2D+D2H timed
  roofline  the generic Pauli-rotation pass (k_pauli_rotation) on a 28-qubit
            state (4 GiB >> L2), algorithmic 32*2^n bytes per pass
  cpu_baseline  the C oracle on this host's cores, bounded sample

Multi-GPU (torchrun): every rank runs its own gradient set (weak scaling, no
data-path collective); the step time is the max over ranks.
`--impl reference` times the CPU oracle (the reference has no implementation
of this path) on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "UCCSD energy evals/sec at 18 qubits (c128); rotation-pass HBM GB/s vs peak"
# ncu --set full of k_pauli_rotation at 28 qubits (profiles/r02/ncu_full_rotation_pass_r02.txt):
# dram__bytes_read.sum + dram__bytes_write.sum per launch (4.295201 + 4.237431 GB);
# algorithmic = 8.589934592 GB
ROT_TRAFFIC_BYTES = 8532632000
UNIT = "evals/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def workload(rank=0):
    from paper_2402_17993_b200 import parameter_shift_set, problems

    P = problems.config_problem(3)
    th0 = P.thetas[0].copy()
    if rank:  # weak scaling: each rank its own seeded theta (same plan)
        th0 = np.array(__import__("paper_2402_17993_b200").uniform_vector(problems.ham_seed(3) + 100 + rank,
                                                                        P.n_gen, -0.1, 0.1))
    rows = np.array(parameter_shift_set(list(th0))).reshape(-1, P.n_gen)
    return P, rows


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, dev):
        self.dev = dev
        self.p = None
        self.out = os.path.join("/tmp", f"ffq_clocks_{os.getpid()}.csv")

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=open(self.out, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            self.p.wait()

    def summary(self):
        try:
            rows = [r.split(", ") for r in open(self.out).read().strip().splitlines()]
            sm = [float(r[1]) for r in rows]
            mx = float(rows[0][2])
            reasons = set()
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for r in rows:
                for nm, v in zip(names, r[5:9]):
                    if v.strip() == "Active":
                        reasons.add(nm)
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                    "samples": len(rows)}
        except Exception as e:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": str(e)[:80]}


def bench_config(world):
    """The `config` dict of both arms (identical, so the driver compares like with like)."""
    return {"workload": "config3: 18 qubits, 10 electrons, 560 UCCSD generators, 9316-term JW "
                        "Hamiltonian; one step = parameter-shift gradient set (1121 energy "
                        "evaluations) per GPU",
            "evals_per_step_per_gpu": 1121, "l2": "flushed (256 MiB write) before every timed step",
            "parallelism": f"replicas x{world} (independent gradient sets)"}


def oracle_workload():
    """Config 3 and its parameter-shift set built by the CPU oracle alone
    (oracle/workload.py): no product import on the reference arm."""
    from oracle import workload as ow

    P = ow.config_problem(3)
    return P, ow.parameter_shift_set(P.thetas[0])


def cpu_oracle_rate(P, rows, n_evals, threads=None):
    from oracle import ffo

    if threads:
        ffo.set_threads(threads)
    t = time.perf_counter()
    es = [P.energy(rows[r]) for r in range(n_evals)]
    dt = time.perf_counter() - t
    return n_evals / dt, es, ffo.get_threads()


def run_reference(args, rank, world):
    if rank != 0:
        return
    P, rows = oracle_workload()
    cores = os.cpu_count() or 1
    evals_per_step = 1
    for _ in range(args.warmup):
        cpu_oracle_rate(P, rows, evals_per_step, cores)
    t = time.perf_counter()
    for s in range(args.steps):
        cpu_oracle_rate(P, rows[s % len(rows):], evals_per_step, cores)
    dt = time.perf_counter() - t
    v = args.steps * evals_per_step / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded h~N(0,1), g~N(0,0.1), theta~U(-0.1,0.1); BASELINE.json config 3)",
        "config": bench_config(args.gpus),
        "path": "CPU oracle (oracle/ffo_oracle.c: SPEC.md restatement, C+OpenMP), dense 2^18 complex128 "
                "state, per-string rotations and term-by-term expectation; inputs from oracle/workload.py",
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{args.steps} x {evals_per_step} evaluation(s) of the config-3 "
                                   "parameter-shift set (rows 0..steps-1)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rot-qubits", type=int, default=28)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sharded", action="store_true", help="skip the sharded-state NCCL leg (child processes)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    args.warmup = max(args.warmup, 3)

    import torch

    # one process per GPU; BENCH_BACKEND=gloo (tests only) lets ranks share a
    # device (no kernel of one rank waits on another's: the legs have no
    # data-path collective) and keeps the scalar collectives on the host
    gpu = local % max(1, torch.cuda.device_count())
    backend = os.environ.get("BENCH_BACKEND", "nccl")
    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(gpu)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(gpu)
    cdev = torch.device("cuda", gpu)

    def max_ranks(v):
        """max over ranks of a host float (device time of the slowest rank)"""
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=cdev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    from paper_2402_17993_b200 import capi

    ctx = capi.Context(gpu)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=cdev)
    P, rows = workload(rank)
    B = rows.shape[0]
    plan = capi.Plan(ctx, P.n_qubits, *P.plan_arrays())
    ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
    th_host = P.plan_thetas(rows)
    th_dev = torch.from_numpy(th_host).to(cdev)
    e_dev = torch.zeros(B, dtype=torch.float64, device=cdev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=cdev)  # 2x L2
    torch.cuda.synchronize()

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def step_device():
        capi.energy_batch_device(ctx, plan, ham, P.hf, B, th_dev.data_ptr(), e_dev.data_ptr())

    def timed(fn, k):
        ms = []
        with torch.cuda.stream(stream):
            for _ in range(k):
                flush.fill_(1)  # L2 flush between timed iterations (untimed)
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                b.synchronize()
                ms.append(a.elapsed_time(b))
        return ms

    for _ in range(args.warmup):
        step_device()
    barrier()
    l0 = ctx.launches()
    with Clocks(gpu) as clk:
        barrier()
        ms = timed(step_device, args.steps)
        barrier()
    launches = ctx.launches() - l0
    tot_ms = sum(ms)
    tot_ms = max_ranks(tot_ms)
    e_first = e_dev.cpu().numpy().copy()
    value = world * B * args.steps / (tot_ms / 1e3)
    # the kernel behind `value`: program statistics for its on-chip roofline
    sector = capi.sector_info(ctx, plan, ham, P.hf)

    # B = 1 latency and B = 64 throughput at 18 qubits (device
    # buffers, CUDA events, L2 flushed before each timed call)
    def batch_call(nb):
        return lambda: capi.energy_batch_device(ctx, plan, ham, P.hf, nb, th_dev.data_ptr(), e_dev.data_ptr())
    b1 = batch_call(1)
    b1()
    ms_b1 = timed(b1, 20)
    b64 = batch_call(64)
    b64()
    ms_b64 = timed(b64, 10)
    # unfused HBM roofline of one evaluation: every generator string
    # a full rotation pass (32 B/amplitude) and every x-group a read pass (16 B)
    n_strings = int(P.plan_arrays()[0][-1])
    n_groups = ham.info()[0]
    unfused_bytes = (32 * n_strings + 16 * n_groups) * 2 ** P.n_qubits
    peak_gbs, _ = peaks()
    unfused_evals = peak_gbs * 1e9 / unfused_bytes
    latency = {"b1_ms": statistics.median(ms_b1), "b64_evals_per_s": 64 / (statistics.median(ms_b64) / 1e3),
               "unfused_roofline_evals_per_s": unfused_evals,
               "x_unfused_roofline": value / world / unfused_evals,
               "unfused_bytes_per_eval": unfused_bytes,
               "note": "unfused roofline = measured HBM peak / (32 B x 2^n per generator string + 16 B x 2^n "
                       "per x-group); label, not a fraction (fusion and on-chip residency pass it)"}

    # e2e: host buffers through ffq_energy_batch (H2D + D2H inside). theta sits in
    # page-locked host memory (a pinned torch tensor viewed as numpy): the library
    # copies from it in place (pageable callers go through its pinned staging buffer)
    th_pinned = torch.from_numpy(th_host).pin_memory()
    th_host_p = th_pinned.numpy()

    def step_host():
        step_host.out = capi.energy_batch(ctx, plan, ham, P.hf, th_host_p)

    step_host()
    barrier()
    ms_e2e = timed(step_host, args.steps)
    barrier()
    tot_e2e = sum(ms_e2e)
    tot_e2e = max_ranks(tot_e2e)
    e2e = world * B * args.steps / (tot_e2e / 1e3)
    assert np.array_equal(step_host.out, e_first), "device and host paths disagree"

    # roofline: the generic rotation pass on a state >> L2
    peak, peak_src = peaks()
    nq = args.rot_qubits
    st = capi.State(ctx, nq, 1)
    st.set_basis(0)
    x, z = (0b1011 << 9), (0b111 << 4)
    for _ in range(3):
        st.rotate(x, z, 0.1)
    ctx.synchronize()
    rot_ms = []
    with torch.cuda.stream(stream):
        for k in range(10):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            st.rotate(x, z, 0.1 * (k % 2 * 2 - 1))
            b.record(stream)
            b.synchronize()
            rot_ms.append(a.elapsed_time(b))
    # the same pass at 18 qubits (north_star's size): 256 rows of 4 MiB = 1 GiB (> L2)
    st18 = capi.State(ctx, 18, 256)
    st18.set_basis(0)
    for _ in range(3):
        st18.rotate(x, z, 0.1)
    ctx.synchronize()
    r18 = []
    with torch.cuda.stream(stream):
        for k in range(10):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            st18.rotate(x, z, 0.1 * (k % 2 * 2 - 1))
            b.record(stream)
            b.synchronize()
            r18.append(a.elapsed_time(b))
    del st18
    r18_avg = statistics.mean(r18[2:])
    rot18 = {"kernel": "k_pauli_rotation", "state_qubits": 18, "rows": 256, "ms_per_pass": r18_avg,
             "achieved_gbs": 256 * 32 * (1 << 18) / (r18_avg / 1e3) / 1e9,
             "frac": 256 * 32 * (1 << 18) / (r18_avg / 1e3) / 1e9 / peak,
             "note": "one rotation pass over 256 batched 18-qubit states (1 GiB, > L2), incl. the API call's cos/sin upload and sync"}
    # fused run: 16 rotations with flip masks in the low 12 qubits (z anywhere),
    # one TMA-staged tile pass (k_rotation_run), then its inverse
    rr = np.random.default_rng(11)
    run_x = rr.integers(1, 1 << 12, size=16, dtype=np.uint64)
    run_z = rr.integers(0, 1 << nq, size=16, dtype=np.uint64)
    run_th = rr.uniform(-1, 1, size=16)
    run_ms = []
    with torch.cuda.stream(stream):
        for k in range(12):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            fwd = k % 2 == 0
            xs, zs, ts = (run_x, run_z, run_th) if fwd else (run_x[::-1].copy(), run_z[::-1].copy(), -run_th[::-1])
            a.record(stream)
            st.rotate_many(xs, zs, ts)  # includes the 16-descriptor upload (1 KiB) and the sync
            b.record(stream)
            b.synchronize()
            run_ms.append(a.elapsed_time(b))
    run_avg = statistics.mean(run_ms[2:])
    rotation_run = {
        "kernel": "k_rotation_run (16 low-qubit rotations per tile pass, 2^12-amplitude TMA tiles)",
        "state_qubits": nq, "rotations_per_run": 16, "ms_per_run": run_avg,
        "hbm_gbs": 32 * (1 << nq) / (run_avg / 1e3) / 1e9,
        "hbm_frac": 32 * (1 << nq) / (run_avg / 1e3) / 1e9 / peak,
        "ms_per_rotation": run_avg / 16,
        "speedup_vs_unfused_passes": 16 * statistics.mean(rot_ms[2:]) / run_avg,
    }
    # gathered tiles: 2 rotations whose flip masks sit on qubits 0-4 and the top 7
    # qubits (the tile is 128 strided 512-byte pieces, one bulk copy each)
    gx = np.array([(int(v) & 31) | ((int(v) >> 5) << (nq - 7)) for v in run_x[:2]], np.uint64)
    gather_ms = []
    with torch.cuda.stream(stream):
        for k in range(12):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            st.rotate_many(gx, run_z[:2], run_th[:2] * (1 if k % 2 == 0 else -1))
            b.record(stream)
            b.synchronize()
            gather_ms.append(a.elapsed_time(b))
    g_avg = statistics.mean(gather_ms[2:])
    rotation_run["gathered_tiles_2_rotations"] = {
        "ms_per_run": g_avg, "hbm_gbs": 32 * (1 << nq) / (g_avg / 1e3) / 1e9,
        "hbm_frac": 32 * (1 << nq) / (g_avg / 1e3) / 1e9 / peak,
        "note": "flip masks on qubits 0-4 and the top 7: tiles of 128 x 512-byte pieces, cp.async.bulk each way"}
    del st
    rot_bytes = 32 * (1 << nq)
    rot_avg = statistics.mean(rot_ms[2:])
    achieved = rot_bytes / (rot_avg / 1e3) / 1e9

    def other_path(env):
        """The same step (same theta rows, device-resident) through another
        execution path selected by FFQ_* knobs read at context creation."""
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        ctx_d = capi.Context(gpu)
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v
        stream_d = torch.cuda.ExternalStream(ctx_d.stream_ptr(), device=cdev)
        plan_d = capi.Plan(ctx_d, P.n_qubits, *P.plan_arrays())
        ham_d = capi.Hamiltonian(ctx_d, P.n_qubits, *P.ham_arrays())
        e_d = torch.zeros(B, dtype=torch.float64, device=cdev)
        f_d = lambda: capi.energy_batch_device(ctx_d, plan_d, ham_d, P.hf, B, th_dev.data_ptr(), e_d.data_ptr())  # noqa: E731
        f_d()
        ctx_d.synchronize()
        with torch.cuda.stream(stream_d):
            a_ev = torch.cuda.Event(enable_timing=True)
            b_ev = torch.cuda.Event(enable_timing=True)
            a_ev.record(stream_d)
            f_d()
            b_ev.record(stream_d)
            b_ev.synchronize()
        out = {"evals_per_s": B / (a_ev.elapsed_time(b_ev) / 1e3),
               "max_abs_diff_vs_value_path": float((e_d - e_dev).abs().max().item())}
        del plan_d, ham_d, ctx_d
        return out

    # secondary: the same step through the complex128 support-closure program
    # (FFQ_SECTOR_REAL=0: full (re, im) amplitudes, 2-CTA clusters), i.e. the
    # c128 arithmetic without the real-amplitude specialisation
    complex_path = other_path({"FFQ_SECTOR_REAL": "0"})
    complex_path["path"] = "k_sector_eval<2,768>: complex128 amplitudes over 2-CTA clusters (DSMEM)"
    # secondary: the support-tracked dense-slab path (FFQ_SECTOR=0): every
    # generator a [chunk][2^n] pass restricted to set support bits, i.e. no
    # support-closure compilation
    dense_path = other_path({"FFQ_SECTOR": "0"})
    dense_path["path"] = "support-tracked [chunk][2^n] slab, CUDA graph of per-generator passes"

    # secondary: BASELINE.json config 2 -- 64 theta vectors x (1 + 2*117) shifts
    # = 15040 evaluations at 12 qubits in one batched call (smem-resident path)
    from paper_2402_17993_b200 import parameter_shift_set, problems as _pb

    P2 = _pb.config_problem(2, batch=64)
    rows2 = np.concatenate([np.array(parameter_shift_set(list(t))).reshape(-1, P2.n_gen) for t in P2.thetas])
    plan2 = capi.Plan(ctx, P2.n_qubits, *P2.plan_arrays())
    ham2 = capi.Hamiltonian(ctx, P2.n_qubits, *P2.ham_arrays())
    th2 = torch.from_numpy(P2.plan_thetas(rows2)).to(cdev)
    e2 = torch.zeros(rows2.shape[0], dtype=torch.float64, device=cdev)
    f2 = lambda: capi.energy_batch_device(ctx, plan2, ham2, P2.hf, rows2.shape[0], th2.data_ptr(),  # noqa: E731
                                         e2.data_ptr())
    for _ in range(2):
        f2()
    ms2 = timed(f2, 3)
    si2 = capi.sector_info(ctx, plan2, ham2, P2.hf)
    config2 = {"evals": int(rows2.shape[0]), "ms_per_call": statistics.mean(ms2),
               "evals_per_s": rows2.shape[0] / (statistics.mean(ms2) / 1e3),
               "path": "%s, one 128-thread CTA per evaluation (eight per SM), support closure of %d amplitudes" % (
                   "k_sector_eval_real" if si2["real_amplitudes"] else "k_sector_eval", si2["closure_size"])}

    # secondary: BASELINE.json config 4 -- FMO batch of 3 monomers (12 q) + 3 dimers
    # (18 q). (a) one evaluation each through the C++ fragment API, fragments
    # sharded over the ranks by cost (shard_by_cost), energies gathered in rank
    # order and assembled with the reference's two-body formula; (b) one FMO
    # gradient step = every fragment's parameter-shift set (3 x 235 + 3 x 1121
    # rows), each fragment's rows split over the ranks (dist.row_range), device-
    # resident theta, max over ranks.
    import paper_2402_17993_b200 as _ff
    from paper_2402_17993_b200 import dist as fdist

    frags = _pb.fmo_fragment_problems()
    dev = _ff.Device(gpu)
    import torch.distributed  # noqa: F401  (fmo_energy imports it: keep the import out of the timed call)
    t_first = time.perf_counter()
    e_fmo2, en = fdist.fmo_energy(frags, 3, lambda fr, r, w: _ff.evaluate_fragments(dev, fr, r, w))
    t_first = time.perf_counter() - t_first
    owners = fdist.fragment_owners(frags, world)
    config4 = {"fragments": len(frags), "e_fmo2": e_fmo2, "first_call_s_incl_compile": t_first,
               "owners": {f.label: int(o) for f, o in zip(frags, owners)},
               "note": "one evaluation per fragment, fragments sharded by cost over the ranks (shard_by_cost)"}
    del dev
    fsets = []
    for lab, Pf in _pb.fmo_fragments().items():
        rf = np.array(parameter_shift_set(list(Pf.thetas[0]))).reshape(-1, Pf.n_gen)
        lo4, hi4 = fdist.row_range(rf.shape[0], rank, world)
        plf = capi.Plan(ctx, Pf.n_qubits, *Pf.plan_arrays())
        hmf = capi.Hamiltonian(ctx, Pf.n_qubits, *Pf.ham_arrays())
        thf = torch.from_numpy(Pf.plan_thetas(rf[lo4:hi4])).to(cdev)
        ef = torch.zeros(max(1, hi4 - lo4), dtype=torch.float64, device=cdev)
        fsets.append((lab, plf, hmf, Pf.hf, hi4 - lo4, thf, ef, rf.shape[0]))

    def fmo_step():
        for _, plf, hmf, hf, nb, thf, ef, _ in fsets:
            if nb:
                capi.energy_batch_device(ctx, plf, hmf, hf, nb, thf.data_ptr(), ef.data_ptr())

    for _ in range(2):
        fmo_step()
    barrier()
    ms4 = timed(fmo_step, 3)
    t4 = statistics.mean(ms4)
    t4 = max_ranks(t4)
    grad = {lab: fdist.gather_rows(ef.cpu().numpy()[:nb], ntot) if dist else ef.cpu().numpy()[:nb]
            for lab, _, _, _, nb, _, ef, ntot in fsets}
    n4 = sum(f[7] for f in fsets)
    config4["gradient_step"] = {
        "evals": n4, "ms_per_step": t4, "evals_per_s": n4 / (t4 / 1e3),
        "e_fmo2_from_step": float(_ff.assemble_fragments(3, {k: float(v[0]) for k, v in grad.items()})),
        "note": "all six fragments' parameter-shift sets, each split over the ranks by rows (dist.row_range), "
                "compiled once, device-resident theta, max over ranks"}
    del fsets

    # SPEC.md:566 (--jobs): fragment VQE runs execute concurrently. One context (own stream)
    # and one host thread per fragment on this GPU, every thread evaluating its fragment's
    # energy (B = 1) `reps` times; wall clock per round of six evaluations, against the same
    # evaluations issued one after another on one context.
    if rank == 0:
        import threading

        reps = 50
        jobs = []
        for lab, Pf in _pb.fmo_fragments().items():
            cj = capi.Context(gpu)
            pj = capi.Plan(cj, Pf.n_qubits, *Pf.plan_arrays())
            hj = capi.Hamiltonian(cj, Pf.n_qubits, *Pf.ham_arrays())
            tj = Pf.plan_thetas()[:1]
            capi.energy_batch(cj, pj, hj, Pf.hf, tj)  # compile
            jobs.append((cj, pj, hj, Pf.hf, tj))

        def serve(job, out, k):
            cj, pj, hj, hf, tj = job
            for _ in range(reps):
                out[k] = capi.energy_batch(cj, pj, hj, hf, tj)[0]

        res = [0.0] * len(jobs)
        t0 = time.perf_counter()
        for k, job in enumerate(jobs):
            serve(job, res, k)
        t_seq = (time.perf_counter() - t0) / reps
        seq = list(res)
        threads = [threading.Thread(target=serve, args=(job, res, k)) for k, job in enumerate(jobs)]
        t0 = time.perf_counter()
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        t_con = (time.perf_counter() - t0) / reps
        config4["concurrent_fragment_jobs"] = {
            "fragments": len(jobs), "ms_per_round_sequential": 1e3 * t_seq, "ms_per_round_concurrent": 1e3 * t_con,
            "same_energies": bool(seq == res),
            "note": "six B = 1 energy evaluations (3 monomers, 3 dimers), one context and host thread per "
                    "fragment on one GPU (SPEC.md:566 --jobs); wall clock incl. H2D/D2H per evaluation"}
        del jobs

    # strong scaling: ONE config-3 gradient set (rank 0's 1121 rows)
    # split over the ranks by dist.row_range, no data-path collective, energies
    # gathered in rank order; must equal the one-GPU energies bit for bit
    P0, rows0 = workload(0)
    lo_s, hi_s = fdist.row_range(rows0.shape[0], rank, world)
    th_s = torch.from_numpy(P0.plan_thetas(rows0[lo_s:hi_s])).to(cdev)
    e_s = torch.zeros(max(1, hi_s - lo_s), dtype=torch.float64, device=cdev)
    f_s = lambda: capi.energy_batch_device(ctx, plan, ham, P0.hf, hi_s - lo_s, th_s.data_ptr(),  # noqa: E731
                                           e_s.data_ptr())
    f_s()
    barrier()
    ms_s = timed(f_s, args.steps)
    t_s = statistics.mean(ms_s)
    t_s = max_ranks(t_s)
    e_all = fdist.gather_rows(e_s.cpu().numpy()[:hi_s - lo_s], rows0.shape[0]) if dist else e_s.cpu().numpy()
    strong = {"evals": int(rows0.shape[0]), "ms_per_step": t_s, "evals_per_s": rows0.shape[0] / (t_s / 1e3),
              "rows_per_rank": hi_s - lo_s,
              "bitwise_equal_to_unsplit": bool(np.array_equal(e_all, e_first)) if rank == 0 else None,
              "note": "scaling strong: one 1121-row gradient set split over the ranks (dist.row_range), "
                      "max over ranks; compare ms_per_step across --gpus N"}

    # secondary: BASELINE.json config 5 (32 qubits, 16 electrons, all singles + the
    # first 2000 doubles, 5000 random Pauli terms) on this GPU: one energy
    # evaluation through the compact real sector layout (1.3 GB instead of 64 GiB)
    # Every rank runs the 8-lane batch on its own seeded theta rows (a config-5 gradient
    # set shards over the GPUs by rows like any batch: weak scaling); rank 0 also times B = 1.
    P5 = _pb.config5_problem()
    t5 = time.perf_counter()
    plan5 = capi.Plan(ctx, P5.n_qubits, *P5.plan_arrays())
    ham5 = capi.Hamiltonian(ctx, P5.n_qubits, *P5.ham_arrays())
    th5 = torch.from_numpy(P5.plan_thetas()).to(cdev)
    e5 = torch.zeros(1, dtype=torch.float64, device=cdev)
    f5 = lambda: capi.energy_batch_device(ctx, plan5, ham5, P5.hf, 1, th5.data_ptr(), e5.data_ptr())  # noqa: E731
    f5()
    ctx.synchronize()
    t5 = time.perf_counter() - t5
    ms5 = timed(f5, 2) if rank == 0 else [0.0]
    # the same evaluation as 8 theta rows interleaved per matrix (one amplitude of
    # 8 evaluations = one 64-byte DRAM atom: passes move algorithmic bytes only)
    rows5 = np.concatenate([P5.thetas, np.random.default_rng(5 + rank).uniform(-0.05, 0.05, size=(7, P5.n_gen))])
    th5b = torch.from_numpy(P5.plan_thetas(rows5)).to(cdev)
    e5b = torch.zeros(8, dtype=torch.float64, device=cdev)
    f5b = lambda: capi.energy_batch_device(ctx, plan5, ham5, P5.hf, 8, th5b.data_ptr(), e5b.data_ptr())  # noqa: E731
    f5b()
    barrier()
    ms5b = timed(f5b, 2)
    t5b = max_ranks(statistics.mean(ms5b))
    config5 = None
    if rank == 0:
        config5 = {"qubits": P5.n_qubits, "generators": P5.n_gen, "terms": len(P5.H), "energy": float(e5.item()),
                   "ms_per_eval": statistics.mean(ms5), "first_call_s_incl_compile": t5,
                   "batch8_ms_per_eval": statistics.mean(ms5b) / 8,
                   "batch8_row0_equals_single": bool(e5b[0].item() == e5.item()),
                   "batch8_all_ranks": {"evals": 8 * world, "ms": t5b, "evals_per_s": 8 * world / (t5b / 1e3),
                                        "note": "every rank its own 8 rows (weak scaling), max over ranks"},
                   "path": "compact real [C(16,8)][C(16,8)][lanes] sector layout, list-driven passes, one GPU "
                           "per evaluation group (no global qubits)"}
    del plan5, ham5

    # sharded state over NCCL: BASELINE config 5's recipe at 26
    # qubits (1 GiB of complex128) split on log2(N) global qubits, one CHILD
    # process per rank (tools/shard_nccl_leg.py: a transport failure cannot take
    # this line with it), half-shard swaps by ncclSend/ncclRecv, max over ranks
    sharded = None
    if world & (world - 1) == 0 and (world == 1 or backend == "nccl") and not args.no_sharded:
        g_sh = world.bit_length() - 1
        ids = [capi.nccl_unique_id().hex() if (rank == 0 and world > 1) else "self"]
        if dist:
            dist.broadcast_object_list(ids, src=0)
        leg = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tools", "shard_nccl_leg.py")
        try:
            r = subprocess.run([sys.executable, leg, "26", str(g_sh), str(rank), ids[0], str(gpu)],
                               capture_output=True, text=True, timeout=300)
            mine = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else {
                "error": (r.stderr or r.stdout)[-300:]}
        except Exception as ex:  # timeout, no output
            mine = {"error": repr(ex)[:300]}
        legs = [mine]
        if dist:
            legs = [None] * world
            dist.all_gather_object(legs, mine)
        if rank == 0:
            bad = [x for x in legs if "error" in x]
            if bad:
                sharded = {"unavailable": bad[0]["error"], "n_gpus": world}
            else:
                sharded = {"n_qubits": 26, "global_qubits": g_sh, "n_gpus": world,
                           "shard_gib": legs[0]["shard_gib"], "swaps_per_eval": legs[0]["swaps_per_eval"],
                           "ms_per_eval": max(x["ms_per_eval"] for x in legs), "energy": legs[0]["energy"],
                           "ranks_agree": all(x["energy"] == legs[0]["energy"] for x in legs),
                           "repeatable": all(x["repeatable"] for x in legs),
                           "note": "sharded path: support-tracked generator passes per shard, expectation batched over "
                                   "support bitmaps, half-shard swaps by ncclSend/ncclRecv; scaling strong: "
                                   "compare ms_per_eval across --gpus N"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_cpu = 2
        OP, orows = oracle_workload()
        assert np.array_equal(orows, rows), "oracle and product parameter-shift sets differ"
        rate, es, cores = cpu_oracle_rate(OP, orows, n_cpu, os.cpu_count())
        parity = max(abs(es[i] - e_first[i]) for i in range(n_cpu))
        rate1, es1, _ = cpu_oracle_rate(OP, orows, 1, 1)  # single-threaded too
        parity = max(parity, abs(es1[0] - e_first[0]))
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{n_cpu} energy evaluations of the config-3 parameter-shift set (C oracle, OpenMP)",
               "parity_max_abs_hartree": parity, "single_thread_value": rate1}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64" if sector["real_amplitudes"] else "c128",
            "dtype_note": ("complex128 semantics; psi(theta) is real for real F and real class sums, so the "
                           "kernel holds the fp64 real parts (imaginary parts identically 0, energies equal to "
                           "the c128 program to <= 1e-12)" if sector["real_amplitudes"] else "complex128"),
            "data": "synthetic (seeded h~N(0,1), g~N(0,0.1), theta~U(-0.1,0.1); BASELINE.json config 3)",
            "config": bench_config(world),
            "path": ("support-closure evaluator: the 15876 amplitudes reachable from |HF> "
                     "(exact for every theta), " + ("real parts only, one CTA per evaluation "
                     "(real F and class sums: psi is real; see DESIGN.md)" if sector["real_amplitudes"]
                     else "complex, %d-CTA cluster" % sector["ctas_per_eval"])),
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(th_host.nbytes),
                    "d2h_bytes_per_step": int(16 * B), "host_buffers": "theta in pinned host memory"},
            "roofline": {"bound": "hbm", "kernel": "k_pauli_rotation (generic rotation pass)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "frac_of_nominal_8tbs": achieved / 8000.0,
                         "traffic": ROT_TRAFFIC_BYTES if nq == 28 else None,
                         "traffic_source": "profiles/r02/ncu_full_rotation_pass_r02.txt (dram read+write per launch, ncu --set full)",
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": rot_bytes, "state_qubits": nq,
                         "avg_launch_ms": rot_avg},
            "gpu_launches": int(launches),
            "secondary": {"config3_latency_and_b64": latency, "config3_complex128_program": complex_path,
                          "config3_dense_slab_path": dense_path,
                          "config2_12q": config2,
                          "config4_fmo": config4, "config3_strong_scaling": strong,
                          "config5_32q": config5, "sharded_state_nccl_26q": sharded,
                          "rotation_run_28q": rotation_run,
                          "rotation_pass_18q_b256": rot18},
            "clocks": clk.summary(),
        }
        # the sector kernel moves no HBM data in the step (theta in, E out, pair
        # tables L2-resident): its bound is shared memory. Algorithmic bytes per
        # evaluation: one amplitude per access (16 B complex, 8 B on the
        # real-amplitude program), a generator pair = 2 loads + 2 stores, an
        # expectation pair = 2 loads; peak = 128 B/clk/SM x SMs x SM clock under
        # load (the Blackwell L1/smem datapath).
        cs = line["clocks"]
        sm_hz = (cs.get("sm_mhz") or 1920) * 1e6
        n_sm = torch.cuda.get_device_properties(gpu).multi_processor_count
        amp_b = 8 if sector["real_amplitudes"] else 16
        # amplitude bytes the program moves through the L1/shared datapath per
        # evaluation: a generator pair 2 loads + 2 stores; a generic expectation
        # pair 2 loads; a block pair 1 load (the anchor is held); a clique
        # lane-row 12 loads (6 + 6 amplitudes for up to 30 pairs)
        generic = sector["expectation_pairs"] - sector["block_pairs"] - sector["clique_pairs"]
        smem_bytes = amp_b * (4 * sector["generator_pairs"] + 2 * generic + sector["block_pairs"]
                              + 12 * sector["clique_lane_rows"])
        smem_ach = smem_bytes * value / world / 1e9
        smem_peak = 128 * n_sm * sm_hz / 1e9
        line["roofline_value_kernel"] = {
            "kernel": "k_sector_eval_real" if sector["real_amplitudes"] else "k_sector_eval", "bound": "smem", "achieved": smem_ach, "peak": smem_peak, "unit": "GB/s",
            "frac": smem_ach / smem_peak, "algorithmic_bytes_per_eval": smem_bytes,
            # round 1's byte model for comparison across rounds: every expectation pair as two
            # amplitude reads (the pairs are the same work; cliques and blocks read fewer bytes for them)
            "pair_model_bytes_per_eval": amp_b * (4 * sector["generator_pairs"] + 2 * sector["expectation_pairs"]),
            "pair_model_frac": amp_b * (4 * sector["generator_pairs"] + 2 * sector["expectation_pairs"])
            * value / world / 1e9 / smem_peak,
            "peak_source": "128 B/clk/SM x %d SMs x median SM clock under load" % n_sm,
            "sector_program": sector}
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
