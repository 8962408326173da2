"""The C ABI boundary (CPU only, no compute calls): libdbtsdf.so loads, exports
exactly the entry points include/dbtsdf.h declares, every one is bound by the
ctypes mirror, the ABI structs have the header's layout, and the oracle library
is separate from the product library."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_2509_20081_b200 import _native

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "dbtsdf.h"


def declared():
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"^DBT_API\s+[\w\s\*]+?\b(dbt_\w+)\s*\(", txt, re.M)))


def test_header_declares_api():
    names = declared()
    assert len(names) >= 25
    for must in ("dbt_grid_create", "dbt_integrate_frame", "dbt_integrate_device", "dbt_popcount",
                 "dbt_signed_distance_field", "dbt_bank_create", "dbt_last_error"):
        assert must in names


def test_library_loads_and_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for name in declared():
        assert hasattr(lib, name), f"{name} declared in dbtsdf.h but not exported"
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    exported = sorted(set(re.findall(r" T (dbt_\w+)", out)))
    assert exported == declared(), "exported dbt_* symbols differ from the header"


def test_ctypes_mirror_binds_every_symbol():
    assert sorted(_native.SIGNATURES) == declared()
    L = _native.lib()
    assert L.dbt_version().decode().startswith("dbtsdf-b200")
    assert isinstance(L.dbt_launch_count(), int)


def test_abi_struct_layout():
    assert ctypes.sizeof(_native.Params) == 24
    assert ctypes.sizeof(_native.Stats) == 80
    txt = HEADER.read_text()
    for f, _ in _native.Params._fields_:
        assert f in txt
    for f, _ in _native.Stats._fields_:
        assert f in txt


def test_engine_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_product_does_not_link_or_import_the_oracle():
    for p in (ROOT / "paper_2509_20081_b200").rglob("*.py"):
        if p.name == "build.py":  # the build recipe compiles the checker, it does not call it
            continue
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p
    out = subprocess.run(["nm", "-D", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "orc_" not in out
