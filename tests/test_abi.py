"""The C-ABI library builds for sm_100a, loads, and exports every symbol
include/mpm.h declares (CPU: no compute calls without a GPU)."""
import ctypes as ct
import os
import re
import subprocess

import pytest

from paper_1910_00935_b200 import build as B
from paper_1910_00935_b200 import mpm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "mpm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mpm_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return mpm.load()


def test_every_declared_symbol_is_exported(lib):
    names = _declared()
    assert len(names) >= 19
    out = subprocess.run(["nm", "-D", "--defined-only", mpm.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (mpm_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(mpm.EXPORTS) == set(names)
    for n in names:
        assert hasattr(lib, n)


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", mpm.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_default_params_host_only(lib):
    p = mpm.mpm_params()
    assert lib.mpm_default_params(3, ct.byref(p)) == 0
    assert p.model == mpm.MODEL_NEOHOOKEAN and p.bound == 3 and abs(p.gravity - 10.0) < 1e-6
    assert lib.mpm_default_params(2, ct.byref(p)) == 0
    assert p.model == mpm.MODEL_FIXED_COROTATED
    assert lib.mpm_default_params(4, ct.byref(p)) == 1  # MPM_ERR_INVALID_ARG


def test_params_struct_matches_header(tmp_path):
    """the ctypes mirror has the header's field order, offsets and size (checked
    against the C compiler's layout of include/mpm.h)"""
    src = open(os.path.join(ROOT, "include", "mpm.h")).read()
    body = src[src.index("typedef struct {", src.index("enum { MPM_LOSS_COM_TARGET")):src.index("} mpm_params;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"\b(?:float|int32_t|int64_t)\s+(\w+)", body)
    assert fields == [f[0] for f in mpm.mpm_params._fields_]
    prog = tmp_path / "layout.c"
    prog.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "mpm.h"\nint main(void){'
                    + "".join(f'printf("%zu ", offsetof(mpm_params, {f}));' for f in fields)
                    + 'printf("%zu", sizeof(mpm_params)); return 0;}\n')
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(prog)])
    got = list(map(int, subprocess.check_output([str(exe)]).split()))
    want = [getattr(mpm.mpm_params, f).offset for f in fields] + [ct.sizeof(mpm.mpm_params)]
    assert got == want


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1910_00935_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                bad = re.findall(r"(?:^|\n)\s*(?:import oracle|from oracle|#include[^\n]*oracle)|oracle_mpm|liboracle", txt)
                assert not bad, (f, bad)


def test_invalid_create_arguments_fail_before_any_device_call(lib):
    """mpm_create validates its arguments on the host (no GPU needed): no particles, a grid
    too small for the 3^d stencil, an unsupported dimension, a non-positive dt or E, or a
    Poisson ratio outside (-1, 1/2) (lambda would be infinite or negative) -> MPM_ERR_INVALID_ARG."""
    h = ct.c_void_p()
    cases = [(0, 64, 3, 1e-3, 25.0, 0.25), (100, 2, 3, 1e-3, 25.0, 0.25), (100, 64, 4, 1e-3, 25.0, 0.25),
             (100, 64, 3, 0.0, 25.0, 0.25), (100, 64, 3, 1e-3, -1.0, 0.25), (100, 64, 3, 1e-3, 25.0, 0.5),
             (100, 64, 2, 1e-3, 25.0, -1.0), (1 << 31, 64, 3, 1e-3, 25.0, 0.25)]
    for args in cases:
        st = lib.mpm_create(*args, ct.byref(h))
        assert st == 1, (args, st)
        assert not h.value
    assert lib.mpm_create(100, 64, 3, 1e-3, 25.0, 0.25, None) == 1
    assert lib.mpm_destroy(None) == 1
