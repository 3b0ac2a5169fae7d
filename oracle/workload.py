"""BASELINE.json configs built from the CPU ORACLE alone (TEST INFRASTRUCTURE).

The reference arm of ``bench.py`` (``--impl reference``) and the CPU baseline
must not touch the product: no ``paper_2402_17993_b200`` import, no product
``.so``. This module restates the synthetic-input recipe on top
of ``oracle/ffo.py`` only:

  ham_seed   = 2402179930 + 1000*config + 10*fragment
  integrals  = ffo.synthetic_integrals(m, ham_seed)          (mt19937_64, Box-Muller)
  H          = ffo.hamiltonian_jw(h, g)
  generators = ffo.build_generators(2m, n_e)
  theta      = ffo.uniform_array(ham_seed + 1, B*P, -w, w)   (batch-major)
  plan       = ffo.magnitude_order(theta[0])
  shift set  = [theta, theta + pi/2 e_0, theta - pi/2 e_0, ...]

``tests/test_golden.py`` holds these inputs to the product's (and to the
committed fixtures): theta and plan bit-identical, Hamiltonian strings
identical and coefficients equal to <= 1e-13 (the two JW expansions sum the
same terms in different orders).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import ffo

SEED_BASE = 2402179930
CONFIGS = {1: (4, 4, 0.1), 2: (6, 6, 0.1), 3: (9, 10, 0.1)}
HALF_PI = 1.5707963267948966


def ham_seed(config: int, fragment: int = 0) -> int:
    return SEED_BASE + 1000 * config + 10 * fragment


@dataclass
class OracleProblem:
    m: int
    n_elec: int
    h: np.ndarray
    g: np.ndarray
    H: "ffo.PauliSum"
    kind: np.ndarray
    idx: np.ndarray
    order: np.ndarray  # plan order (int32), by |theta row 0|
    thetas: np.ndarray  # [batch][n_gen], canonical generator order

    @property
    def n_qubits(self):
        return 2 * self.m

    @property
    def n_gen(self):
        return len(self.kind)

    def energy(self, theta):
        """energy_trotter of one canonical-order theta row."""
        return ffo.energy_trotter(self.n_qubits, self.n_elec, self.kind, self.idx, self.order,
                                  np.ascontiguousarray(theta, np.float64), self.H)[0]


def config_problem(config: int, batch: int = 1, fragment: int = 0) -> OracleProblem:
    m, ne, hw = CONFIGS[config]
    seed = ham_seed(config, fragment)
    h, g = ffo.synthetic_integrals(m, seed)
    H = ffo.hamiltonian_jw(h, g)
    kind, idx = ffo.build_generators(2 * m, ne)
    th = ffo.uniform_array(seed + 1, batch * len(kind), -hw, hw).reshape(batch, len(kind))
    order = ffo.magnitude_order(th[0])
    return OracleProblem(m, ne, h, g, H, kind, idx, order, th)


def parameter_shift_set(theta) -> np.ndarray:
    """[1 + 2P][P]: theta, then theta +- pi/2 e_k for k = 0..P-1 (+ before -)."""
    th = np.asarray(theta, np.float64)
    P = len(th)
    rows = np.repeat(th[None, :], 1 + 2 * P, axis=0)
    k = np.arange(P)
    rows[1 + 2 * k, k] += HALF_PI
    rows[2 + 2 * k, k] -= HALF_PI
    return rows
