"""The C-ABI library: loads, exports every symbol include/luxb200.h declares,
ctypes struct layouts equal the C layouts, and the host-side BVH builder
(no GPU needed) reproduces the reference-built trees bit for bit."""
from __future__ import annotations

import ctypes as C
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden_scene

HEADER = ROOT / "include" / "luxb200.h"


def declared_symbols() -> list[str]:
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(lt_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_exports_all_symbols():
    from paper_2407_19977_b200 import _lib
    from paper_2407_19977_b200.build import build
    build()
    handle = C.CDLL(str(_lib.LIB_PATH))
    syms = declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(handle, s)]
    assert missing == []
    assert set(syms) == set(_lib.SIGNATURES)
    assert _lib.lib().lt_abi_version() == 2


def test_struct_layouts_match_header(tmp_path):
    from paper_2407_19977_b200 import _lib
    structs = {"lt_scene_desc": _lib.SceneDesc, "lt_render_params": _lib.RenderParams,
               "lt_render_stats": _lib.RenderStats, "lt_scene_info": _lib.SceneInfo}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for field, _ in py._fields_:
            lines.append(f'printf("{cname}.{field} %zu\\n", offsetof({cname}, {field}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["/usr/bin/gcc", str(src), "-o", str(exe)], check=True)
    out = dict(line.rsplit(" ", 1) for line in subprocess.check_output([str(exe)]).decode()
               .strip().splitlines())
    for cname, py in structs.items():
        assert int(out[cname]) == C.sizeof(py), cname
        for field, _ in py._fields_:
            assert int(out[f"{cname}.{field}"]) == getattr(py, field).offset, f"{cname}.{field}"


def test_errors_are_reported():
    from paper_2407_19977_b200 import _lib
    lib = _lib.lib()
    n = C.c_int64()
    z = np.zeros((0, 3))
    rc = lib.lt_build_bvh(_lib.ptr(z, C.c_double), _lib.ptr(z, C.c_double),
                          _lib.ptr(z, C.c_double), 0, 4, 12, None, None, None, None, None, None,
                          None, C.byref(n), C.byref(n), C.byref(n))
    assert rc == _lib.LT_ERR_INVALID
    with pytest.raises(ValueError, match="empty scene"):
        from paper_2407_19977_b200 import TriangleBuffer, build_bvh
        build_bvh(TriangleBuffer(*[np.zeros((0, 3))] * 6))


@pytest.mark.parametrize("name", ["floor", "shell", "glossy", "sphere2k", "dup", "cornell_c1",
                                  "cornell_c2", "sphere20k"])
def test_host_bvh_build_matches_reference(name):
    """build_bvh (csrc/lt_bvh_build.cpp) == luxtrace.build_bvh, bit for bit."""
    from paper_2407_19977_b200 import build_bvh
    g = golden_scene(name)
    b = build_bvh(g.triangles, device=None)
    assert np.array_equal(b.bounds_min, g["bvh_bounds_min"])
    assert np.array_equal(b.bounds_max, g["bvh_bounds_max"])
    assert np.array_equal(b.left_child, g["bvh_left"])
    assert np.array_equal(b.right_child, g["bvh_right"])
    assert np.array_equal(b.first_triangle, g["bvh_first"])
    assert np.array_equal(b.triangle_count, g["bvh_count"])
    assert np.array_equal(b.triangle_order, g["bvh_order"])
    assert b.stats.node_count == len(g["bvh_left"])
    assert b.stats.node_count == 2 * b.stats.leaf_count - 1


def test_host_bvh_leaf_size_and_single_triangle():
    from paper_2407_19977_b200 import TriangleBuffer, build_bvh
    g = golden_scene("sphere2k")
    big = build_bvh(g.triangles, leaf_size=12, device=None)
    assert int(big.triangle_count.max()) <= 12
    one = TriangleBuffer(np.array([[0.0, 0, 0]]), np.array([[1.0, 0, 0]]), np.array([[0.0, 1, 0]]),
                         *[np.array([[0.0, 0, 1]])] * 3)
    b = build_bvh(one, device=None)
    assert b.stats.node_count == 1 and b.stats.leaf_count == 1
    assert int(b.triangle_count[0]) == 1
