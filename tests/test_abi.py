"""C-ABI library: loads, exports every symbol include/qapsa.h declares, and
validates its arguments before touching a device (no GPU needed)."""
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1208_2675_b200 import qapsa as Q
from qap_inputs import taixxa, start_perm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qapsa.h")


def _header_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(qap_[a-z_]+)\s*\(", txt)))


def test_library_builds_and_loads():
    L = Q.lib()
    assert os.path.exists(Q.LIB_PATH)
    assert Q.qap_version() == 1
    assert L is Q.lib()


def test_every_declared_symbol_is_exported():
    declared = _header_functions()
    assert len(declared) >= 14
    assert set(declared) == set(Q.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", Q.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (qap_\w+)", out))
    missing = set(declared) - exported
    assert not missing, missing


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", Q.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_status_strings():
    for code, name in Q.STATUS.items():
        assert Q.qap_status_str(code) == name


def _expect(status, fn):
    with pytest.raises(Q.QapError) as ei:
        fn()
    assert ei.value.status == status, str(ei.value)


def test_create_validation_errors():
    A, B = taixxa(8, 1)
    p0 = start_perm(8, 1)
    _expect(1, lambda: Q.qap_create(A[:1, :1], B[:1, :1], p0[:1]))          # n < 2
    bad = A.copy(); bad[0, 1] += 1
    _expect(3, lambda: Q.qap_create(bad, B, p0))                               # asymmetric
    diag = B.copy(); diag[2, 2] = 1
    _expect(3, lambda: Q.qap_create(A, diag, p0))                              # nonzero diagonal
    neg = A.copy(); neg[0, 1] = neg[1, 0] = -1
    _expect(3, lambda: Q.qap_create(neg, B, p0))                               # negative entry
    _expect(2, lambda: Q.qap_create(A, B, np.zeros(8, np.int32)))             # not a permutation
    big = np.full((8, 8), 65535, np.int32); np.fill_diagonal(big, 0)
    _expect(4, lambda: Q.qap_create(big, big, p0))                            # overflow bound


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU error path")
def test_no_cpu_fallback_without_gpu():
    A, B = taixxa(8, 1)
    _expect(7, lambda: Q.qap_create(A, B, start_perm(8, 1)))


def test_null_ctx_is_an_error():
    _expect(1, lambda: Q.qap_delta_init(None))
