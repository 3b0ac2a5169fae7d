"""ctypes binding of the CPU ORACLE (``oracle/_build/libffo_oracle.so``).

TEST INFRASTRUCTURE ONLY. Importable from ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` legs, where it is the
checker or the timed CPU baseline -- never the product path. The product
package (``paper_2402_17993_b200``) must not import this module.

Each wrapper mirrors one SPEC operation (``/root/reference/SPEC.md`` lines
cited in ``ffo_oracle.h``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libffo_oracle.so")
_lib = None

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


def build() -> str:
    """Compile the oracle (gcc, seconds)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
        os.path.join(_HERE, "ffo_oracle.c")
    ):
        build()
    L = C.CDLL(_SO)
    P = C.c_void_p
    sig = {
        "ffo_mt64_nth": (C.c_uint64, [C.c_uint64, C.c_int]),
        "ffo_uniform_array": (None, [C.c_uint64, C.c_int, C.c_double, C.c_double, _f64p]),
        "ffo_synthetic_integrals": (None, [C.c_int, C.c_uint64, C.c_double, C.c_double, _f64p, _f64p]),
        "ffo_pauli_mul": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                    C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "ffo_psum_new": (P, [C.c_int]),
        "ffo_psum_free": (None, [P]),
        "ffo_psum_size": (C.c_int, [P]),
        "ffo_psum_nqubits": (C.c_int, [P]),
        "ffo_psum_get": (None, [P, _u64p, _u64p, _f64p, _f64p]),
        "ffo_psum_from_arrays": (P, [C.c_int, C.c_int, _u64p, _u64p, _f64p, _f64p]),
        "ffo_jw_add_product": (None, [P, C.c_int, _i32p, _i32p, C.c_double, C.c_double]),
        "ffo_psum_simplify": (None, [P]),
        "ffo_hamiltonian_jw": (P, [C.c_int, _f64p, _f64p, C.c_double]),
        "ffo_build_generators": (C.c_int, [C.c_int, C.c_int, P, P]),
        "ffo_generator_image": (P, [C.c_int, C.c_int, _i32p]),
        "ffo_magnitude_order": (None, [C.c_int, _f64p, _i32p]),
        "ffo_set_threads": (None, [C.c_int]),
        "ffo_get_threads": (C.c_int, []),
        "ffo_hf_state": (None, [C.c_int, C.c_uint64, _f64p]),
        "ffo_apply_pauli_rotation": (None, [C.c_int, _f64p, C.c_uint64, C.c_uint64, C.c_double]),
        "ffo_expectation": (None, [C.c_int, _f64p, P, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "ffo_energy_trotter": (C.c_double, [C.c_int, C.c_int, C.c_int, _i32p, _i32p, _i32p, _f64p, P,
                                            P, C.POINTER(C.c_double)]),
        "ffo_energy_fermionic": (C.c_double, [C.c_int, C.c_int, _f64p, _f64p, C.c_double, C.c_int,
                                              _i32p, _i32p, _i32p, _f64p, P]),
        "ffo_fmo_assemble": (C.c_double, [C.c_int, C.c_int, _f64p, C.c_int, _f64p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


class PauliSum:
    """Oracle-side Pauli sum (owning handle)."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ffo_psum_free(self.h)
            self.h = None

    @classmethod
    def from_terms(cls, n, x, z, c):
        x = np.ascontiguousarray(x, np.uint64)
        z = np.ascontiguousarray(z, np.uint64)
        c = np.asarray(c, np.complex128)
        return cls(lib().ffo_psum_from_arrays(n, len(x), x, z, np.ascontiguousarray(c.real),
                                              np.ascontiguousarray(c.imag)))

    @property
    def n_qubits(self):
        return lib().ffo_psum_nqubits(self.h)

    def __len__(self):
        return lib().ffo_psum_size(self.h)

    def terms(self):
        n = len(self)
        x = np.zeros(n, np.uint64); z = np.zeros(n, np.uint64)
        cr = np.zeros(n); ci = np.zeros(n)
        lib().ffo_psum_get(self.h, x, z, cr, ci)
        return x, z, cr + 1j * ci


def mt64_nth(seed: int, nth: int) -> int:
    return int(lib().ffo_mt64_nth(seed, nth))


def uniform_array(seed, count, lo, hi):
    out = np.zeros(count)
    lib().ffo_uniform_array(seed, count, lo, hi, out)
    return out


def synthetic_integrals(m, seed, sigma_h=1.0, sigma_g=0.1):
    h = np.zeros(m * m); g = np.zeros(m ** 4)
    lib().ffo_synthetic_integrals(m, seed, sigma_h, sigma_g, h, g)
    return h.reshape(m, m), g.reshape(m, m, m, m)


def pauli_mul(n, x1, z1, x2, z2):
    x3 = C.c_uint64(); z3 = C.c_uint64()
    k = lib().ffo_pauli_mul(n, x1, z1, x2, z2, C.byref(x3), C.byref(z3))
    return k, x3.value, z3.value


def jw_product(n, ops, coef=1.0 + 0j):
    """JW image of coef * prod(ops); ops = [(index, is_dagger), ...] left to right."""
    s = lib().ffo_psum_new(n)
    idx = np.array([o[0] for o in ops], np.int32)
    dg = np.array([1 if o[1] else 0 for o in ops], np.int32)
    lib().ffo_jw_add_product(s, len(ops), idx, dg, coef.real, coef.imag)
    lib().ffo_psum_simplify(s)
    return PauliSum(s)


def hamiltonian_jw(h, g, e_const=0.0):
    m = h.shape[0]
    return PauliSum(lib().ffo_hamiltonian_jw(m, np.ascontiguousarray(h, np.float64).ravel(),
                                             np.ascontiguousarray(g, np.float64).ravel(), e_const))


def build_generators(n_so, n_e):
    n = lib().ffo_build_generators(n_so, n_e, None, None)
    kind = np.zeros(n, np.int32); idx = np.zeros(4 * n, np.int32)
    lib().ffo_build_generators(n_so, n_e, kind.ctypes.data, idx.ctypes.data)
    return kind, idx.reshape(n, 4)


def generator_image(n_so, kind, idx4):
    return PauliSum(lib().ffo_generator_image(n_so, int(kind), np.ascontiguousarray(idx4, np.int32)))


def magnitude_order(amps):
    amps = np.ascontiguousarray(amps, np.float64)
    out = np.zeros(len(amps), np.int32)
    lib().ffo_magnitude_order(len(amps), amps, out)
    return out


def set_threads(n):
    lib().ffo_set_threads(n)


def get_threads():
    return lib().ffo_get_threads()


def hf_state(n, occ_bits):
    psi = np.zeros(2 << n)
    lib().ffo_hf_state(n, occ_bits, psi)
    return psi.view(np.complex128)


def apply_pauli_rotation(n, psi, x, z, theta):
    buf = np.ascontiguousarray(psi, np.complex128).view(np.float64).copy()
    lib().ffo_apply_pauli_rotation(n, buf, x, z, theta)
    return buf.view(np.complex128)


def expectation(n, psi, H: PauliSum):
    buf = np.ascontiguousarray(psi, np.complex128).view(np.float64)
    re = C.c_double(); im = C.c_double()
    lib().ffo_expectation(n, buf, H.h, C.byref(re), C.byref(im))
    return complex(re.value, im.value)


def energy_trotter(n_so, n_e, kind, idx, plan, amps, H: PauliSum, want_state=False):
    kind = np.ascontiguousarray(kind, np.int32)
    idx = np.ascontiguousarray(idx, np.int32).ravel()
    plan = np.ascontiguousarray(plan, np.int32)
    amps = np.ascontiguousarray(amps, np.float64)
    im = C.c_double()
    psi = np.zeros(2 << n_so) if want_state else None
    e = lib().ffo_energy_trotter(n_so, n_e, len(kind), kind, idx, plan, amps, H.h,
                                 psi.ctypes.data if want_state else None, C.byref(im))
    if want_state:
        return e, im.value, psi.view(np.complex128)
    return e, im.value


def energy_fermionic(h, g, n_e, kind, idx, plan, amps, e_const=0.0, want_state=False):
    m = h.shape[0]
    psi = np.zeros(2 << (2 * m)) if want_state else None
    e = lib().ffo_energy_fermionic(
        m, n_e, np.ascontiguousarray(h, np.float64).ravel(), np.ascontiguousarray(g, np.float64).ravel(),
        e_const, len(kind), np.ascontiguousarray(kind, np.int32),
        np.ascontiguousarray(idx, np.int32).ravel(), np.ascontiguousarray(plan, np.int32),
        np.ascontiguousarray(amps, np.float64), psi.ctypes.data if want_state else None)
    if want_state:
        return e, psi.view(np.complex128)
    return e


def fmo_assemble(n_fragments, monomers, dimers):
    mono = np.ascontiguousarray(monomers, np.float64)
    dim = np.ascontiguousarray(dimers, np.float64)
    return lib().ffo_fmo_assemble(n_fragments, len(mono), mono, len(dim), dim)
