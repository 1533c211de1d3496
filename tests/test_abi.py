"""The C-ABI library loads and exports every entry point its headers declare;
without a GPU the device path refuses loudly (no CPU fallback exists)."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADERS = [ROOT / "include/ngdb/ngdb_cuda.h", ROOT / "include/ngdb/ngdb_host.h"]


def declared(path):
    text = path.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ngdb_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header", HEADERS, ids=lambda p: p.name)
def test_every_declared_symbol_is_exported(header):
    from paper_2602_21597_b200._native import LIB_PATH
    lib = C.CDLL(str(LIB_PATH))
    names = declared(header)
    assert len(names) >= 10
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_signatures_cover_headers():
    from paper_2602_21597_b200._native import SIGNATURES
    names = set(declared(HEADERS[0])) | set(declared(HEADERS[1]))
    assert names <= set(SIGNATURES), sorted(names - set(SIGNATURES))


def test_oracle_header_symbols():
    import oracle as O
    names = re.findall(r"\b(oracle_[a-z0-9_]+)\s*\(",
                       re.sub(r"/\*.*?\*/", "", (ROOT / "oracle/include/oracle.h").read_text(), flags=re.S))
    assert all(hasattr(O.lib, n) for n in names)


def test_no_device_fails_loudly():
    from conftest import HAS_GPU
    if HAS_GPU:
        pytest.skip("a GPU is present")
    import paper_2602_21597_b200 as m
    from paper_2602_21597_b200._native import NgdbError
    with pytest.raises(NgdbError) as e:
        m.Engine("gqe", 10, 2, dim=8, n_neg=2)
    assert e.value.kind == "NoDevice"
