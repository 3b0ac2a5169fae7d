"""SPEC.md:298-305 FCIDUMP interchange and SPEC.md:459 state dump (host only)."""
import os
import struct

import numpy as np
import pytest

import paper_2402_17993_b200 as ff
from paper_2402_17993_b200 import problems


def test_fcidump_round_trip_is_lossless(tmp_path):
    h, g = ff.synthetic_integrals(6, problems.ham_seed(2))
    p = str(tmp_path / "c2.fcidump")
    ff.write_fcidump(p, h, g, 6, e_const=-1.25)
    h2, g2, e2, ne, ms2 = ff.read_fcidump(p)
    assert np.array_equal(h, h2) and np.array_equal(g, g2)  # 17 significant digits: bitwise
    assert e2 == -1.25 and ne == 6 and ms2 == 0
    # the qubit image of the read-back Hamiltonian is identical term by term
    a = ff.qubit_hamiltonian(h, g, 6, -1.25).arrays()
    b = ff.qubit_hamiltonian(h2, g2, ne, e2).arrays()
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


def test_fcidump_zero_two_electron_part_has_only_one_electron_lines(tmp_path):
    h, _ = ff.synthetic_integrals(3, 5)
    g = np.zeros((3, 3, 3, 3))
    p = str(tmp_path / "h.fcidump")
    ff.write_fcidump(p, h, g, 2)
    body = [ln.split() for ln in open(p).read().split("&END")[1].strip().splitlines()]
    assert all(int(t[3]) == 0 and int(t[4]) == 0 for t in body)
    assert len(body) == 3 * 4 // 2 + 1  # h_ij (i >= j) + the constant line


def test_fcidump_header_and_8fold_symmetry(tmp_path):
    h, g = ff.synthetic_integrals(4, problems.ham_seed(1))
    p = str(tmp_path / "c1.fcidump")
    ff.write_fcidump(p, h, g, 4)
    txt = open(p).read()
    assert "NORB=4" in txt and "NELEC=4" in txt
    lines = txt.split("&END")[1].strip().splitlines()
    two = [t for t in (ln.split() for ln in lines) if int(t[3]) != 0]
    assert len(two) == 4 * 5 // 2 * (4 * 5 // 2 + 1) // 2  # unique (ij|kl), ij >= kl


def test_fcidump_malformed_raises_parse_error(tmp_path):
    p = str(tmp_path / "bad.fcidump")
    with open(p, "w") as f:
        f.write(" &FCI NORB=2,NELEC=2,\n &END\n0.5 1 1 0\n")
    with pytest.raises(ff.ParseError):
        ff.read_fcidump(p)
    with open(p, "w") as f:
        f.write(" &FCI NELEC=2,\n &END\n")
    with pytest.raises(ff.ParseError):
        ff.read_fcidump(p)


def test_state_dump_format(tmp_path):
    rng = np.random.default_rng(3)
    a = rng.standard_normal(32) + 1j * rng.standard_normal(32)
    p = str(tmp_path / "psi.bin")
    ff.write_state_dump(p, 5, list(a))
    raw = open(p, "rb").read()
    assert len(raw) == 8 + 32 * 16 and struct.unpack("<q", raw[:8])[0] == 5
    assert np.array_equal(np.frombuffer(raw[8:], "<c16"), a)  # LE complex doubles, qubit 0 = LSB order
    n, b = ff.read_state_dump(p)
    assert n == 5 and np.array_equal(np.array(b), a)
    with open(p, "ab") as f:
        f.write(b"x")
    with pytest.raises(ff.ParseError):
        ff.read_state_dump(p)


def test_cli_ham_and_usage_errors(tmp_path, capsys):
    from paper_2402_17993_b200 import cli

    out = str(tmp_path / "c1.fcidump")
    assert cli.main(["ham", "--config", "1", "--out", out]) == 0
    rep = __import__("json").loads(capsys.readouterr().out)
    assert rep["records"][0]["norb"] == 4 and rep["provenance"]["config_sha256"]
    h, g, e, ne, _ = ff.read_fcidump(out)
    P = problems.config_problem(1)
    assert np.array_equal(h, P.h) and np.array_equal(g, P.g) and ne == 4
    assert cli.main(["nonsense"]) == 1  # usage error -> exit 1
    capsys.readouterr()
    assert cli.main(["energy", "--fcidump", str(tmp_path / "missing")]) == 1
