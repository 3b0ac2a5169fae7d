"""Config 4 (FMO fragment batch) on the GPU through the C++ facade:
3 monomers at 12 qubits + 3 dimers at 18 qubits, assembled with the
reference's two-body formula (fmo.cpp:28-48)."""
import numpy as np
import pytest

import paper_2402_17993_b200 as ff
from paper_2402_17993_b200 import problems

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fmo():
    dev = ff.Device(0)
    frags = problems.fmo_fragment_problems()
    return dev, frags, ff.evaluate_fragments(dev, frags)


def test_fmo_fragments_vs_oracle(fmo, oracle):
    dev, frags, energies = fmo
    probs = problems.fmo_fragments()
    for lab in ("1", "2", "3", "21"):
        P = probs[lab]
        x, z, c = P.ham_arrays()
        H = oracle.PauliSum.from_terms(P.n_qubits, x, z, c)
        kind, idx = oracle.build_generators(P.n_qubits, P.n_elec)
        ref = oracle.energy_trotter(P.n_qubits, P.n_elec, kind, idx, np.array(P.plan.order, np.int32),
                                    P.thetas[0], H)[0]
        assert abs(energies[lab] - ref) <= 1e-10, lab


def test_fmo_sharded_equals_single_and_assembles(fmo):
    dev, frags, energies = fmo
    for world in (2, 4, 8):
        union = {}
        for r in range(world):
            part = ff.evaluate_fragments(dev, frags, r, world)
            assert not (set(part) & set(union))
            union.update(part)
        assert union == energies  # bitwise: same device path per fragment
    e = ff.assemble_fragments(3, energies)
    mono = sum(energies[k] for k in ("1", "2", "3"))
    dim = sum(energies[k] for k in ("21", "31", "32"))
    assert abs(e - (dim - mono)) <= 1e-12  # N_f = 3: E = sum E_IJ - sum E_I
    fmo2 = mono + sum(energies[a + b] - energies[a] - energies[b] for a, b in (("2", "1"), ("3", "1"), ("3", "2")))
    assert abs(e - fmo2) <= 1e-10  # FMO2 form (BASELINE.json config 4)
