"""Seeded synthetic workloads of BASELINE.json's configs (DESIGN.md pins them).

Each problem bundles the JW qubit Hamiltonian, the UCCSD generators, the
magnitude-ordered plan and the theta vectors, all built by the C++ host API.
Seeds: ham_seed = 2402179930 + 1000*config + 10*fragment; theta_seed = ham_seed + 1.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import (build_generators, hf_bits, magnitude_order, qubit_hamiltonian, reduce_two_qubits,
               reduce_two_qubits_basis, synthetic_integrals, uniform_vector)

SEED_BASE = 2402179930

# config -> (spatial orbitals m, electrons, theta half-width)
CONFIGS = {1: (4, 4, 0.1), 2: (6, 6, 0.1), 3: (9, 10, 0.1)}


def ham_seed(config: int, fragment: int = 0) -> int:
    return SEED_BASE + 1000 * config + 10 * fragment


@dataclass
class Problem:
    name: str
    m: int
    n_elec: int
    h: np.ndarray
    g: np.ndarray
    H: object  # PauliSum
    gens: list
    plan: object  # TrotterPlan
    thetas: np.ndarray  # [batch][n_gen], canonical generator order
    seed: int
    extra: dict = field(default_factory=dict)
    mapping: str = "jw"  # "jw" or "scbkt" (two-qubit reduction)
    images: list = None  # scbkt: reduced generator images by canonical id

    @property
    def n_qubits(self):
        return 2 * self.m - (2 if self.mapping == "scbkt" else 0)

    @property
    def n_gen(self):
        return len(self.gens)

    @property
    def hf(self):
        if self.mapping == "scbkt":
            return reduce_two_qubits_basis(hf_bits(self.n_elec), 2 * self.m)
        return hf_bits(self.n_elec)

    def plan_thetas(self, thetas=None):
        """[batch][n_gen] in plan (execution) order."""
        t = self.thetas if thetas is None else np.atleast_2d(thetas)
        return np.ascontiguousarray(t[:, np.asarray(self.plan.order)])

    def plan_arrays(self):
        """Flat C-ABI arrays of the plan: term_off, x, z, c (execution order)."""
        off = [0]; xs = []; zs = []; cs = []
        for gid in self.plan.order:
            x, z, c = (self.images[gid] if self.images is not None else self.gens[gid].image).arrays()
            xs.append(x); zs.append(z); cs.append(c)
            off.append(off[-1] + len(x))
        return (np.array(off, np.int64), np.concatenate(xs).astype(np.uint64),
                np.concatenate(zs).astype(np.uint64), np.concatenate(cs))

    def ham_arrays(self):
        return self.H.arrays()


def make_problem(m: int, n_elec: int, seed: int, batch: int = 1, theta_hw: float = 0.1,
                 name: str = "", mapping: str = "jw") -> Problem:
    """mapping "scbkt": the Hamiltonian and every generator image go through
    reduce_two_qubits (2m - 2 qubits); the Trotter energy is mapping
    independent (each generator's strings commute, so its exponential is exact)."""
    h, g = synthetic_integrals(m, seed)
    return problem_from_integrals(h, g, n_elec, seed=seed, batch=batch, theta_hw=theta_hw,
                                  name=name or f"m{m}e{n_elec}", mapping=mapping)


def problem_from_integrals(h, g, n_elec: int, e_const: float = 0.0, seed: int = SEED_BASE, batch: int = 1,
                           theta_hw: float = 0.1, name: str = "", mapping: str = "jw") -> Problem:
    """A problem from spatial integrals (e.g. read_fcidump); theta rows seeded
    from `seed` + 1 as for the synthetic configs."""
    h = np.ascontiguousarray(h, np.float64)
    g = np.ascontiguousarray(g, np.float64)
    m = h.shape[0]
    H = qubit_hamiltonian(h, g, n_elec, e_const)
    gens = build_generators(2 * m, n_elec)
    th = np.array(uniform_vector(seed + 1, batch * len(gens), -theta_hw, theta_hw)).reshape(batch, len(gens))
    plan = magnitude_order(gens, list(th[0]), 2 * m)
    images = None
    if mapping == "scbkt":
        na, nb = (n_elec + 1) // 2, n_elec // 2  # |HF>: lowest spin orbitals, interleaved
        H = reduce_two_qubits(H, 2 * m, na, nb)
        images = [reduce_two_qubits(gn.image, 2 * m, na, nb) for gn in gens]
    elif mapping != "jw":
        raise ValueError(f"unknown mapping {mapping!r}")
    return Problem(name or f"m{m}e{n_elec}", m, n_elec, h, g, H, gens, plan, th, seed, mapping=mapping,
                   images=images, extra={"e_const": e_const})


def config_problem(config: int, batch: int = 1, fragment: int = 0, mapping: str = "jw") -> Problem:
    m, ne, hw = CONFIGS[config]
    return make_problem(m, ne, ham_seed(config, fragment), batch, hw, name=f"config{config}", mapping=mapping)


def fmo_fragments():
    """Config 4: monomers "1".."3" (12 qubits, 6 e) and dimers "21","31","32"
    (18 qubits, 10 e), each with its own seed."""
    frags = {}
    for f in (1, 2, 3):
        frags[str(f)] = make_problem(6, 6, ham_seed(4, f), name=f"monomer{f}")
    for k, lab in enumerate(("21", "31", "32")):
        frags[lab] = make_problem(9, 10, ham_seed(4, 10 + k), name=f"dimer{lab}")
    return frags


def fmo_fragment_problems():
    """Config 4 as FragmentProblem objects (C++ FMO batch input)."""
    from . import FragmentProblem

    out = []
    for label, P in fmo_fragments().items():
        out.append(FragmentProblem(label, P.H, P.plan, P.hf, list(P.thetas[0])))
    return out


def config5_problem(n_doubles: int = 2000, n_terms: int = 5000, n_qubits: int = 32, n_elec: int = 16):
    """BASELINE.json config 5: all singles + the first `n_doubles` doubles in
    canonical generator order (pinned reading of "first 2000 seeded doubles"),
    theta ~ U(-0.05, 0.05), H = `n_terms` seeded random {I,X,Y,Z}^n strings with
    real c ~ N(0, 0.1)."""
    from . import random_pauli_hamiltonian

    seed = ham_seed(5)
    gens_all = build_generators(n_qubits, n_elec)
    singles = [g for g in gens_all if g.exc.kind == 1]
    doubles = [g for g in gens_all if g.exc.kind == 2][:n_doubles]
    gens = singles + doubles
    th = np.array(uniform_vector(seed + 1, len(gens), -0.05, 0.05)).reshape(1, len(gens))
    plan = magnitude_order(gens, list(th[0]), n_qubits)
    H = random_pauli_hamiltonian(n_qubits, n_terms, seed + 2, 0.1)
    return Problem(f"config5_{n_qubits}q", n_qubits // 2, n_elec, None, None, H, gens, plan, th, seed)
