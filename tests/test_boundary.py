"""The C ABI: library loads, exports every symbol include/sgiga.h declares,
descriptor layout, error mapping (no GPU compute here)."""
from __future__ import annotations

import ctypes as ct
import re

import pytest

from conftest import ROOT
from paper_1707_09598_b200 import _lib
from paper_1707_09598_b200.errors import (DeviceError, EmptyInteriorError, InvalidGeometryError,
                                          LinearSolveError)


def declared_symbols():
    text = (ROOT / "include" / "sgiga.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sgiga_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"libsgiga.so does not export {n}"
    assert set(names) == set(_lib.EXPORTED)


def test_descriptor_layout_matches_header():
    # pointer-aligned C layout: 5 ints, 4 pointers, int (+pad), 3 pointers, 4 pointers, 2 ints
    assert ct.sizeof(_lib.ProblemDesc) == 5 * 4 + 4 + 4 * 8 + 8 + 3 * 8 + 4 * 8 + 8
    assert _lib.ProblemDesc.levels.offset == 24


def test_status_codes_map_to_reference_exceptions(monkeypatch):
    monkeypatch.setattr(_lib, "last_error", lambda: "msg")
    for code, exc in ((-1, ValueError), (-2, InvalidGeometryError), (-3, LinearSolveError),
                      (-4, EmptyInteriorError), (-5, DeviceError), (-7, KeyError)):
        with pytest.raises(exc):
            _lib.check(code)
    _lib.check(0)


def test_create_rejects_bad_descriptor_without_gpu():
    from paper_1707_09598_b200.analysis import BenchmarkProblem, constant_one
    from paper_1707_09598_b200.geometry import unit_hypercube
    from paper_1707_09598_b200.pipeline import make_desc
    from paper_1707_09598_b200.scheduler import make_spec

    prob = BenchmarkProblem("p5", unit_hypercube(2), constant_one, 5, 4)   # degree 5 > device max
    desc, keep = make_desc(make_spec((((1, 1), 1),), prob))
    h = ct.c_void_p()
    assert _lib.load().sgiga_create(ct.byref(desc), None, ct.byref(h)) == _lib.SGIGA_ERR_VALUE
    assert "degree" in _lib.last_error()


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle."""
    pkg = ROOT / "paper_1707_09598_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f
