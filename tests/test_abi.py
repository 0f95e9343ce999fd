"""C-ABI boundary: libifgfb200 loads, exports every entry point that
include/ifgfb.h declares, the ctypes struct layouts equal the C layouts, and
compute calls fail loudly (no CPU fallback) when no GPU is present."""

import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2408_02274_b200 import _lib
from paper_2408_02274_b200.build import build

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "ifgfb.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ifgfb_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    build()
    return _lib.load()


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) <= set(_lib.EXPORTS), "ctypes table out of date"


def test_abi_version(lib):
    assert lib.ifgfb_abi_version() == _lib.ABI_VERSION == 8


STRUCTS = {
    "ifgfb_tree_desc": _lib.TreeDesc,
    "ifgfb_level_desc": _lib.LevelDesc,
    "ifgfb_emit_desc": _lib.EmitDesc,
    "ifgfb_accum_desc": _lib.AccumDesc,
    "ifgfb_surface_desc": _lib.SurfaceDesc,
    "ifgfb_near_desc": _lib.NearDesc,
    "ifgfb_level_part": _lib.LevelPart,
    "ifgfb_partition_desc": _lib.PartitionDesc,
    "ifgfb_rank_desc": _lib.RankDesc,
    "ifgfb_cone_level_desc": _lib.ConeLevelDesc,
    "ifgfb_cone_parent_desc": _lib.ConeParentDesc,
    "ifgfb_accum_types_desc": _lib.AccumTypesDesc,
}


def test_struct_layouts_match_c(tmp_path):
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "ifgfb.h"',
           "int main(void) {"]
    for cname, py in STRUCTS.items():
        src.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            src.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    src.append("return 0; }")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(c), "-o", str(exe)],
                   check=True)
    got = dict(line.split() for line in subprocess.run(
        [str(exe)], check=True, capture_output=True, text=True).stdout.splitlines())
    for cname, py in STRUCTS.items():
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    pts = np.zeros((4, 3))
    perm = np.arange(4, dtype=np.int64)
    td = _lib.TreeDesc(4, 3, 3, 5, _lib.dptr(pts), _lib.iptr(perm))
    h = ctypes.c_void_p()
    rc = lib.ifgfb_plan_create(td, h)
    assert rc == -2
    assert b"no CPU fallback" in lib.ifgfb_last_error()
    with pytest.raises(RuntimeError):
        _lib.check(rc, "ifgfb_plan_create")


def test_bad_orders_rejected(lib):
    pts = np.zeros((4, 3))
    perm = np.arange(4, dtype=np.int64)
    td = _lib.TreeDesc(4, 3, 4, 5, _lib.dptr(pts), _lib.iptr(perm))
    h = ctypes.c_void_p()
    rc = lib.ifgfb_plan_create(td, h)
    assert rc == -1
    with pytest.raises(ValueError):
        _lib.check(rc, "ifgfb_plan_create")


def test_product_does_not_import_oracle():
    pkg = ROOT / "paper_2408_02274_b200"
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert "import oracle" not in text and "from oracle" not in text, f
