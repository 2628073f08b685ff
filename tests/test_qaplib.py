"""QAPLIB file I/O (paper_1208_2675_b200/qaplib.py), host side only."""
import itertools
import os

import numpy as np
import pytest

import oracle as O
from paper_1208_2675_b200 import qaplib
from qap_inputs import taixxa

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_dat_and_sln_roundtrip(tmp_path):
    A, B = taixxa(17, 3, hi=60000)
    f = str(tmp_path / "x.dat")
    qaplib.write_dat(f, A, B)
    A2, B2 = qaplib.read_dat(f)
    np.testing.assert_array_equal(A, A2)
    np.testing.assert_array_equal(B, B2)
    p = np.random.default_rng(1).permutation(17).astype(np.int32)
    g = str(tmp_path / "x.sln")
    qaplib.write_sln(g, 12345, p)
    n, cost, p2 = qaplib.read_sln(g)
    assert (n, cost) == (17, 12345)
    np.testing.assert_array_equal(p, p2)


def test_tiny_fixture_optimum_by_brute_force():
    """tests/golden/qaplib_tiny4.{dat,sln}: a hand-written 4x4 instance and its optimum, checked
    by enumerating all 24 permutations with Eq.(1) summed here and by the oracle's cost."""
    A, B = qaplib.read_dat(os.path.join(GOLD, "qaplib_tiny4.dat"))
    n, cost, p = qaplib.read_sln(os.path.join(GOLD, "qaplib_tiny4.sln"))
    assert n == 4 and A.shape == (4, 4)
    eq1 = lambda q: int(sum(int(A[i, j]) * int(B[q[i], q[j]]) for i in range(4) for j in range(4)))
    assert min(eq1(q) for q in itertools.permutations(range(4))) == cost == eq1(p)
    assert O.cost(A, B, p) == cost


def test_malformed_files_raise(tmp_path):
    f = tmp_path / "bad.dat"
    f.write_text("3\n1 2 3\n")
    with pytest.raises(ValueError):
        qaplib.read_dat(str(f))
    g = tmp_path / "bad.sln"
    g.write_text("3 10\n1 1 2\n")
    with pytest.raises(ValueError):
        qaplib.read_sln(str(g))


@pytest.mark.parametrize("text,kind", [("1\n0\n0\n", "size"), ("2\n0 -1 -1 0\n0 1 1 0\n", "domain"),
                                       ("2\n0 1 1 x\n0 1 1 0\n", "parse")])
def test_spec_error_kinds(tmp_path, text, kind):
    """SPEC's error classes: n < 2 is a size error, negative entries a domain error, a bad token
    a parse error that names its position."""
    f = tmp_path / "e.dat"
    f.write_text(text)
    with pytest.raises(qaplib.QaplibError) as ei:
        qaplib.read_dat(str(f))
    assert ei.value.kind == kind
    if kind == "parse":
        assert "token 4" in str(ei.value)
