"""fragfield B200: the UCCSD state-vector hot path of arXiv 2402.17993 on sm_100a.

Python mirror of the C++ operator API (include/fragfield/*.hpp), which in turn
drives the C-ABI of ``lib/libfragfield_cuda.so`` (include/fragfield_cuda.h).
The operation names follow the reference SPEC (``/root/reference/SPEC.md``):
``jordan_wigner``, ``build_generators``, ``magnitude_order``, ``hf_state`` (as
``Statevector.set_basis``), ``apply_pauli_rotation``, ``expectation``,
``energy_trotter``, ``vqe_minimize``.

There is no CPU fallback: importing this package without the built native
libraries raises ImportError, and device calls without a GPU raise DeviceError.
"""
from __future__ import annotations

import os as _os

_LIB = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "lib")

try:
    from .lib import _fragfield as _native  # noqa: F401
except ImportError as e:  # pragma: no cover - exercised only on a broken install
    raise ImportError(
        "paper_2402_17993_b200: native library not built "
        "(run `python paper_2402_17993_b200/_build.py`): " + str(e)
    ) from e

from .lib._fragfield import (  # noqa: E402,F401
    ContractViolation,
    ParseError,
    ConvergenceError,
    Device,
    DeviceError,
    DeviceHamiltonian,
    DevicePlan,
    Excitation,
    FragmentProblem,
    Generator,
    OptimizerOptions,
    OptimizeResult,
    PauliString,
    PauliSum,
    Statevector,
    TrotterPlan,
    assemble_fragments,
    ao_to_mo,
    assemble_two_body,
    bfgs_minimize,
    build_generators,
    dimer_labels,
    energy_batch,
    energy_exact,
    energy_trotter,
    evaluate_fragments,
    GroundState,
    lanczos_ground,
    exact_gradient_from_energies,
    freeze_core,
    fragment_cost,
    exact_gradient_set,
    hf_bits,
    jordan_wigner,
    magnitude_order,
    neldermead_minimize,
    reduce_two_qubits,
    reduce_two_qubits_basis,
    read_fcidump,
    read_state_dump,
    write_fcidump,
    write_state_dump,
    parameter_shift_set,
    pauli_mul,
    powell_minimize,
    qubit_hamiltonian,
    random_pauli_hamiltonian,
    shard_by_cost,
    synthetic_integrals,
    uniform_vector,
    vqe_bfgs,
    vqe_device,
)


def vqe_minimize(objective, x0, optimizer: str = "powell", opts=None):
    """derivative-free VQE driver (Powell or Nelder-Mead)."""
    opts = opts or OptimizerOptions()
    if optimizer == "powell":
        return powell_minimize(objective, list(x0), opts)
    if optimizer == "neldermead":
        return neldermead_minimize(objective, list(x0), opts)
    raise ContractViolation("vqe_minimize: optimizer must be 'powell' or 'neldermead'")


def native_library_path() -> str:
    return _os.path.join(_LIB, "libfragfield_cuda.so")


__all__ = [n for n in dir() if not n.startswith("_")]
