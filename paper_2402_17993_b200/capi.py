"""ctypes binding of the C-ABI in include/fragfield_cuda.h.

This is the binding a reference-side maintainer would write:
plain pointers and sizes, return codes mapped to exceptions. The GPU parity
tests and bench.py's end-to-end leg call the hot path through it.
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

from . import ContractViolation, DeviceError, native_library_path

FFQ_OK, FFQ_EINVAL, FFQ_ENONHERMITIAN, FFQ_ECUDA, FFQ_ENOMEM, FFQ_ENCCL, FFQ_ENODEV = 0, -1, -2, -3, -4, -5, -6

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_vp = C.c_void_p

_SIGS = {
    "ffq_version": (C.c_int, []),
    "ffq_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "ffq_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "ffq_ctx_destroy": (C.c_int, [_vp]),
    "ffq_ctx_synchronize": (C.c_int, [_vp]),
    "ffq_last_error": (C.c_char_p, [_vp]),
    "ffq_ctx_kernel_launches": (C.c_int64, [_vp]),
    "ffq_ctx_stream": (C.c_int, [_vp, C.POINTER(_vp)]),
    "ffq_ham_upload": (C.c_int, [_vp, C.c_int, C.c_int64, _u64p, _u64p, _f64p, _f64p, C.POINTER(_vp)]),
    "ffq_ham_destroy": (C.c_int, [_vp]),
    "ffq_ham_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "ffq_plan_upload": (C.c_int, [_vp, C.c_int, C.c_int, _i64p, _u64p, _u64p, _f64p, _f64p, C.POINTER(_vp)]),
    "ffq_plan_destroy": (C.c_int, [_vp]),
    "ffq_plan_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ffq_energy_batch": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_int, _f64p, _f64p]),
    "ffq_energy_batch_device": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_int, _vp, _vp, _vp]),
    "ffq_energy_prepare": (C.c_int, [_vp, _vp, _vp, C.c_uint64]),
    "ffq_state_alloc": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(_vp)]),
    "ffq_state_free": (C.c_int, [_vp]),
    "ffq_state_set_basis": (C.c_int, [_vp, C.c_uint64]),
    "ffq_state_upload": (C.c_int, [_vp, _f64p]),
    "ffq_state_download": (C.c_int, [_vp, _f64p]),
    "ffq_state_apply_pauli_rotation": (C.c_int, [_vp, C.c_uint64, C.c_uint64, C.c_double]),
    "ffq_state_apply_pauli_rotations": (C.c_int, [_vp, C.c_int, _u64p, _u64p, _f64p]),
    "ffq_rotation_groups": (C.c_int, [C.c_int, C.c_int, C.c_int, _u64p, _i32p, _i32p, _i32p, _u64p,
                                      np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS"), _i32p,
                                      C.POINTER(C.c_int32)]),
    "ffq_state_apply_plan": (C.c_int, [_vp, _vp, _f64p]),
    "ffq_state_expectation": (C.c_int, [_vp, _vp, _f64p, _f64p]),
    "ffq_state_device_ptr": (C.c_int, [_vp, C.POINTER(_vp)]),
    "ffq_shard_create": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(_vp)]),
    "ffq_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "ffq_shard_create_nccl": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(_vp)]),
    "ffq_shard_destroy": (C.c_int, [_vp]),
    "ffq_shard_energy": (C.c_int, [_vp, _vp, _vp, C.c_uint64, _f64p, C.POINTER(C.c_double)]),
    "ffq_shard_download": (C.c_int, [_vp, _f64p]),
    "ffq_shard_info": (C.c_int, [_vp, C.POINTER(C.c_int), np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")]),
    "ffq_shard_schedule": (C.c_int, [C.c_int, C.c_int, C.c_int, _i64p, _u64p, _u64p, _f64p, _f64p,
                                     np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"),
                                     np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"),
                                     C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ffq_shard_schedule_steps": (C.c_int, [C.c_int, C.c_int, C.c_int, _i64p, _u64p, _u64p, _f64p, _f64p,
                                           np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"),
                                           np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"),
                                           C.POINTER(C.c_int), C.POINTER(C.c_int),
                                           np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"), C.c_int]),
    "ffq_lanczos_ground": (C.c_int, [_vp, _vp, C.c_uint64, C.c_double, C.c_int, C.POINTER(C.c_double),
                                     C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ffq_energy_exact": (C.c_int, [_vp, _vp, _vp, C.c_uint64, _f64p, C.c_double, C.POINTER(C.c_double)]),
    "ffq_ham_compile_stats": (C.c_int, [C.c_int, C.c_int64, _u64p, _u64p, _f64p, _f64p, _i64p]),
    "ffq_plan_compile_stats": (C.c_int, [C.c_int, C.c_int, _i64p, _u64p, _u64p, _f64p, _f64p, _i64p]),
    "ffq_sector_emulate": (C.c_int, [C.c_int, C.c_int, _i64p, _u64p, _u64p, _f64p, _f64p, C.c_int64, _u64p, _u64p,
                                     _f64p, _f64p, C.c_uint64, _f64p, _f64p]),
    "ffq_compact_emulate": (C.c_int, [C.c_int, C.c_int, _i64p, _u64p, _u64p, _f64p, _f64p, C.c_int64, _u64p, _u64p,
                                      _f64p, _f64p, C.c_uint64, _f64p, _f64p]),
    "ffq_sector_info": (C.c_int, [_vp, _vp, _vp, C.c_uint64, _i64p]),
    "ffq_sector_state": (C.c_int, [_vp, _vp, _vp, C.c_uint64, _f64p, _f64p, C.POINTER(C.c_double)]),
    "ffq_multi_create": (C.c_int, [np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"), C.c_int,
                                   C.POINTER(_vp)]),
    "ffq_multi_destroy": (C.c_int, [_vp]),
    "ffq_multi_device_count": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "ffq_multi_last_error": (C.c_char_p, [_vp]),
    "ffq_multi_problem_upload": (C.c_int, [_vp, C.c_int, C.c_int, _i64p, _u64p, _u64p, _f64p, _f64p, C.c_int64,
                                           _u64p, _u64p, _f64p, _f64p, C.POINTER(C.c_int)]),
    "ffq_multi_energy_batch": (C.c_int, [_vp, C.c_int, C.c_uint64, C.c_int, _f64p, _f64p]),
    "ffq_multi_energy_units": (C.c_int, [_vp, C.c_int, np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"),
                                         _u64p, np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"),
                                         C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                         np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(native_library_path())
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def header_symbols(path=None):
    """Every function the public header declares."""
    path = path or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "include", "fragfield_cuda.h")
    src = open(path).read()
    return sorted(set(re.findall(r"\b(ffq_[a-z0-9_]+)\s*\(", src)))


def check(rc, ctx=None):
    if rc == FFQ_OK:
        return
    msg = lib().ffq_last_error(ctx).decode()
    if rc in (FFQ_EINVAL, FFQ_ENONHERMITIAN):
        raise ContractViolation(msg)
    raise DeviceError(f"[{rc}] {msg}")


def _terms(x, z, c):
    c = np.asarray(c, np.complex128)
    return (np.ascontiguousarray(x, np.uint64), np.ascontiguousarray(z, np.uint64),
            np.ascontiguousarray(c.real), np.ascontiguousarray(c.imag))


def ham_compile_stats(n, x, z, c):
    x, z, re_, im = _terms(x, z, c)
    st = np.zeros(8, np.int64)
    check(lib().ffq_ham_compile_stats(n, len(x), x, z, re_, im, st))
    keys = ["groups", "terms", "classes", "active_patterns", "work_items", "pair_visits",
            "class_evals", "bytes_read"]
    return dict(zip(keys, st.tolist()))


def plan_compile_stats(n, off, x, z, c):
    x, z, re_, im = _terms(x, z, c)
    off = np.ascontiguousarray(off, np.int64)
    st = np.zeros(6, np.int64)
    check(lib().ffq_plan_compile_stats(n, len(off) - 1, off, x, z, re_, im, st))
    keys = ["fused", "string_ops", "pattern_pairs", "pair_updates", "bytes", "ops"]
    return dict(zip(keys, st.tolist()))


def sector_emulate(n, plan_arrays, ham_arrays, hf_bits, psi):
    """Host emulation of the real one-CTA sector program's expectation on the
    real state psi (no GPU); returns the energy and the layout statistics."""
    off, px, pz, pc = plan_arrays
    px, pz, pre, pim = _terms(px, pz, pc)
    hx, hz, hre, him = _terms(*ham_arrays)
    off = np.ascontiguousarray(off, np.int64)
    psi = np.ascontiguousarray(psi, np.float64)
    out = np.zeros(11)
    check(lib().ffq_sector_emulate(n, len(off) - 1, off, px, pz, pre, pim, len(hx), hx, hz, hre, him, hf_bits, psi,
                                   out))
    keys = ["energy", "closure_size", "slots", "product", "block_pairs", "exp_pairs", "generic_rows", "units",
            "clique_pairs", "clique_conflicts", "table_violations"]
    return dict(zip(keys, out.tolist()))


def compact_emulate(n, plan_arrays, ham_arrays, hf_bits, theta_plan_order):
    """Host emulation of the compact real sector program (no GPU): energy of one
    theta row and the list statistics (ffq_compact_emulate)."""
    off, px, pz, pc = plan_arrays
    px, pz, pre, pim = _terms(px, pz, pc)
    hx, hz, hre, him = _terms(*ham_arrays)
    off = np.ascontiguousarray(off, np.int64)
    th = np.ascontiguousarray(theta_plan_order, np.float64).ravel()
    out = np.zeros(8)
    check(lib().ffq_compact_emulate(n, len(off) - 1, off, px, pz, pre, pim, len(hx), hx, hz, hre, him, hf_bits, th,
                                    out))
    keys = ["energy", "eligible", "alpha_strings", "beta_strings", "generator_pairs", "term_pairs", "violations",
            "term_groups"]
    return dict(zip(keys, out.tolist()))


class Context:
    """One device + stream (ffq_ctx_t)."""

    def __init__(self, device=0):
        h = _vp()
        check(lib().ffq_ctx_create(device, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            try:
                _lib.ffq_ctx_destroy(self.h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None

    __del__ = close

    def launches(self):
        return lib().ffq_ctx_kernel_launches(self.h)

    def stream_ptr(self):
        p = _vp()
        check(lib().ffq_ctx_stream(self.h, C.byref(p)), self.h)
        return p.value or 0

    def synchronize(self):
        check(lib().ffq_ctx_synchronize(self.h), self.h)


class Hamiltonian:
    def __init__(self, ctx: Context, n, x, z, c):
        self.ctx = ctx
        x, z, re_, im = _terms(x, z, c)
        h = _vp()
        check(lib().ffq_ham_upload(ctx.h, n, len(x), x, z, re_, im, C.byref(h)), ctx.h)
        self.h = h

    def info(self):
        g = C.c_int(); t = C.c_int64(); cl = C.c_int64()
        check(lib().ffq_ham_info(self.h, C.byref(g), C.byref(t), C.byref(cl)))
        return g.value, t.value, cl.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            try:
                _lib.ffq_ham_destroy(self.h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None


class Plan:
    def __init__(self, ctx: Context, n, off, x, z, c):
        self.ctx = ctx
        x, z, re_, im = _terms(x, z, c)
        off = np.ascontiguousarray(off, np.int64)
        self.n_gen = len(off) - 1
        h = _vp()
        check(lib().ffq_plan_upload(ctx.h, n, self.n_gen, off, x, z, re_, im, C.byref(h)), ctx.h)
        self.h = h

    def info(self):
        f = C.c_int(); s = C.c_int()
        check(lib().ffq_plan_info(self.h, C.byref(f), C.byref(s)))
        return f.value, s.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            try:
                _lib.ffq_plan_destroy(self.h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None


def energy_batch(ctx: Context, plan: Plan, ham: Hamiltonian, hf_bits: int, theta):
    theta = np.ascontiguousarray(theta, np.float64)
    batch = theta.shape[0] if theta.ndim == 2 else 1
    out = np.zeros(batch)
    check(lib().ffq_energy_batch(ctx.h, plan.h, ham.h, hf_bits, batch, theta.ravel(), out), ctx.h)
    return out


def energy_batch_device(ctx: Context, plan: Plan, ham: Hamiltonian, hf_bits: int, batch, theta_ptr,
                        e_ptr, im_ptr=None):
    check(lib().ffq_energy_batch_device(ctx.h, plan.h, ham.h, hf_bits, batch, theta_ptr, e_ptr, im_ptr),
          ctx.h)


SECTOR_INFO_KEYS = ("closure_size", "ctas_per_eval", "generator_pairs", "expectation_pairs",
                    "expectation_rows", "cluster_barrier_steps", "split_mask", "chunk_buffer_amplitudes",
                    "real_amplitudes", "block_pairs", "slots", "clique_pairs", "clique_warp_tasks",
                    "clique_conflicts", "clique_lane_rows")


def energy_prepare(ctx: Context, plan: Plan, ham: Hamiltonian, hf_bits: int):
    """Compile and cache the program energy_batch runs for these handles (thread-safe for distinct plans)."""
    check(lib().ffq_energy_prepare(ctx.h, plan.h, ham.h, hf_bits), ctx.h)


def sector_state(ctx: Context, plan: Plan, ham: Hamiltonian, hf_bits: int, theta, n_qubits: int):
    """(psi[2^n] complex128 in natural order, energy) of one evaluation of the
    real-amplitude sector program (ffq_sector_state); theta in plan order."""
    th = np.ascontiguousarray(theta, np.float64).ravel()
    psi = np.zeros(2 << n_qubits)
    e = C.c_double()
    check(lib().ffq_sector_state(ctx.h, plan.h, ham.h, hf_bits, th, psi, C.byref(e)), ctx.h)
    return psi.view(np.complex128), e.value


def sector_info(ctx: Context, plan: Plan, ham: Hamiltonian, hf_bits: int) -> dict:
    """Statistics of the support-closure program energy_batch runs (ffq_sector_info)."""
    out = np.zeros(15, np.int64)
    check(lib().ffq_sector_info(ctx.h, plan.h, ham.h, hf_bits, out), ctx.h)
    return dict(zip(SECTOR_INFO_KEYS, (int(v) for v in out)))


class State:
    def __init__(self, ctx: Context, n, batch=1):
        self.ctx, self.n, self.batch = ctx, n, batch
        h = _vp()
        check(lib().ffq_state_alloc(ctx.h, n, batch, C.byref(h)), ctx.h)
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            try:
                _lib.ffq_state_free(self.h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None

    def set_basis(self, bits):
        check(lib().ffq_state_set_basis(self.h, bits), self.ctx.h)

    def upload(self, psi):
        buf = np.ascontiguousarray(psi, np.complex128).reshape(-1)
        if buf.size != self.batch << self.n:
            raise ContractViolation("state size mismatch")
        check(lib().ffq_state_upload(self.h, buf.view(np.float64)), self.ctx.h)

    def download(self):
        out = np.zeros(2 * (self.batch << self.n))
        check(lib().ffq_state_download(self.h, out), self.ctx.h)
        return out.view(np.complex128).reshape(self.batch, 1 << self.n)

    def rotate(self, x, z, theta):
        check(lib().ffq_state_apply_pauli_rotation(self.h, x, z, theta), self.ctx.h)

    def rotate_many(self, x, z, theta):
        """e^{i theta_r P_r} for r = 0, 1, ... in order (low-qubit runs fused in tiles)."""
        x = np.ascontiguousarray(x, np.uint64); z = np.ascontiguousarray(z, np.uint64)
        th = np.ascontiguousarray(theta, np.float64)
        if not (x.shape == z.shape == th.shape) or x.ndim != 1:
            raise ContractViolation("x, z, theta must be 1-D arrays of one length")
        check(lib().ffq_state_apply_pauli_rotations(self.h, len(x), x, z, th), self.ctx.h)

    def apply_plan(self, plan: Plan, theta):
        check(lib().ffq_state_apply_plan(self.h, plan.h, np.ascontiguousarray(theta, np.float64).ravel()),
              self.ctx.h)

    def expectation(self, ham: Hamiltonian):
        re_ = np.zeros(self.batch); im = np.zeros(self.batch)
        check(lib().ffq_state_expectation(self.h, ham.h, re_, im), self.ctx.h)
        return re_ + 1j * im

    def device_ptr(self):
        p = _vp()
        check(lib().ffq_state_device_ptr(self.h, C.byref(p)))
        return p.value


def rotation_groups(n, t, x):
    """Host-only: how ffq_state_apply_pauli_rotations cuts flip masks x on n
    qubits for tile bits t -> (run_of, group_of, cx, run_q, basis [G][3], piv [G][3])."""
    x = np.ascontiguousarray(x, np.uint64)
    m = len(x)
    run_of = np.zeros(m, np.int32); group_of = np.zeros(m, np.int32); cx = np.zeros(m, np.int32)
    run_q = np.zeros(m, np.uint64)
    basis = np.zeros(3 * max(m, 1), np.uint32); piv = np.zeros(3 * max(m, 1), np.int32)
    ng = C.c_int32(0)
    check(lib().ffq_rotation_groups(n, t, m, x, run_of, group_of, cx, run_q, basis, piv, C.byref(ng)))
    g = ng.value
    return run_of, group_of, cx, run_q, basis[:3 * g].reshape(g, 3), piv[:3 * g].reshape(g, 3)


def shard_schedule(n, n_global, off, x, z, c):
    """Host-only swap schedule: (init_perm, final_perm, n_swaps, n_steps)."""
    x, z, re_, im = _terms(x, z, c)
    off = np.ascontiguousarray(off, np.int64)
    ip = np.zeros(n, np.int32); fp = np.zeros(n, np.int32)
    ns = C.c_int(); st = C.c_int()
    check(lib().ffq_shard_schedule(n, n_global, len(off) - 1, off, x, z, re_, im, ip, fp, C.byref(ns), C.byref(st)))
    return ip, fp, ns.value, st.value


def shard_schedule_steps(n, n_global, off, x, z, c):
    """(init_perm, final_perm, steps[n_steps][4]) with steps = (kind, gpos, lpos, generator column)."""
    x, z, re_, im = _terms(x, z, c)
    off = np.ascontiguousarray(off, np.int64)
    ip = np.zeros(n, np.int32); fp = np.zeros(n, np.int32)
    ns = C.c_int(); st = C.c_int()
    cap = 4 * (len(off) - 1) + 64 * n
    steps = np.zeros(4 * cap, np.int32)
    check(lib().ffq_shard_schedule_steps(n, n_global, len(off) - 1, off, x, z, re_, im, ip, fp, C.byref(ns),
                                         C.byref(st), steps, cap))
    return ip, fp, steps[: 4 * st.value].reshape(-1, 4)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().ffq_nccl_unique_id(buf))
    return buf.raw


class ShardedState:
    """A state split on n_global physical qubits over 2^n_global ranks.
    nccl_id=None: every rank on this context's device (group mode);
    else this process is `rank` of an NCCL communicator."""

    def __init__(self, ctx: Context, n, n_global, rank=None, nccl_id=None):
        self.ctx, self.n, self.g = ctx, n, n_global
        h = _vp()
        if nccl_id is None:
            check(lib().ffq_shard_create(ctx.h, n, n_global, C.byref(h)), ctx.h)
        else:
            check(lib().ffq_shard_create_nccl(ctx.h, n, n_global, rank, nccl_id, C.byref(h)), ctx.h)
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            try:
                _lib.ffq_shard_destroy(self.h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None

    def energy(self, plan: Plan, ham: Hamiltonian, hf_bits, theta):
        e = C.c_double()
        check(lib().ffq_shard_energy(self.h, plan.h, ham.h, hf_bits,
                                     np.ascontiguousarray(theta, np.float64).ravel(), C.byref(e)), self.ctx.h)
        return e.value

    def download(self):
        out = np.zeros(2 << self.n)
        check(lib().ffq_shard_download(self.h, out), self.ctx.h)
        return out.view(np.complex128)

    def info(self):
        sw = C.c_int(); perm = np.zeros(self.n, np.int32)
        check(lib().ffq_shard_info(self.h, C.byref(sw), perm))
        return sw.value, perm


def lanczos_ground(ctx: Context, ham: Hamiltonian, hf_bits, tol=1e-10, max_iter=500):
    """CAS-CI ground energy in the Krylov space of |hf>."""
    e = C.c_double(); it = C.c_int(); dim = C.c_int()
    check(lib().ffq_lanczos_ground(ctx.h, ham.h, hf_bits, tol, max_iter, C.byref(e), C.byref(it), C.byref(dim)),
          ctx.h)
    return e.value, it.value, dim.value


def energy_exact(ctx: Context, plan: Plan, ham: Hamiltonian, hf_bits, theta, tol=1e-12):
    """Trotter-free UCCSD energy; theta in plan order."""
    e = C.c_double()
    check(lib().ffq_energy_exact(ctx.h, plan.h, ham.h, hf_bits, np.ascontiguousarray(theta, np.float64).ravel(),
                                 tol, C.byref(e)), ctx.h)
    return e.value


class Multi:
    """One context per device (ffq_multi_*): independent units sharded over the
    devices of one node by host threads, no collective; results equal the
    one-device call bit for bit."""

    def __init__(self, devices):
        devs = np.ascontiguousarray(devices, np.int32)
        h = _vp()
        self._lib = lib()
        rc = self._lib.ffq_multi_create(devs, len(devs), C.byref(h))
        if rc != 0:
            check(rc)
        self.h = h

    def _check(self, rc):
        if rc == FFQ_OK:
            return
        msg = self._lib.ffq_multi_last_error(self.h).decode()
        if rc in (FFQ_EINVAL, FFQ_ENONHERMITIAN):
            raise ContractViolation(msg)
        raise DeviceError(f"[{rc}] {msg}")

    def __del__(self):
        if getattr(self, "h", None):
            self._lib.ffq_multi_destroy(self.h)
            self.h = None

    def device_count(self):
        n = C.c_int()
        self._check(self._lib.ffq_multi_device_count(self.h, C.byref(n)))
        return n.value

    def upload(self, n, plan_arrays, ham_arrays):
        off, px, pz, pc = plan_arrays
        px, pz, pre, pim = _terms(px, pz, pc)
        hx, hz, hre, him = _terms(*ham_arrays)
        pid = C.c_int()
        self._check(self._lib.ffq_multi_problem_upload(self.h, n, len(off) - 1, np.ascontiguousarray(off, np.int64),
                                                       px, pz, pre, pim, len(hx), hx, hz, hre, him, C.byref(pid)))
        return pid.value

    def energy_batch(self, problem, hf_bits, theta):
        th = np.ascontiguousarray(np.atleast_2d(theta), np.float64)
        e = np.zeros(th.shape[0])
        self._check(self._lib.ffq_multi_energy_batch(self.h, problem, hf_bits, th.shape[0], th, e))
        return e

    def energy_units(self, problems_, hf_bits, thetas):
        ths = [np.ascontiguousarray(np.atleast_2d(t), np.float64) for t in thetas]
        es = [np.zeros(t.shape[0]) for t in ths]
        n = len(ths)
        tp = (C.c_void_p * n)(*[t.ctypes.data for t in ths])
        ep = (C.c_void_p * n)(*[e.ctypes.data for e in es])
        dev = np.zeros(n, np.int32)
        self._check(self._lib.ffq_multi_energy_units(
            self.h, n, np.ascontiguousarray(problems_, np.int32), np.ascontiguousarray(hf_bits, np.uint64),
            np.array([t.shape[0] for t in ths], np.int32), tp, ep, dev))
        return es, dev.tolist()
