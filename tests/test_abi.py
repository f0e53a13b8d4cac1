"""C-ABI checks that need no GPU: the library was built for sm_100a, loads,
exports every function include/dts.h declares, and the binding's struct
layouts match the header (compiled with gcc here)."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dts.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:dts_status|size_t|int32_t|const char\*)\s+(dts_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2402_03106_b200 import dts
    lib = dts.lib_handle()
    names = _declared()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(dts.EXPORTED)
    assert dts.abi_version() == 2
    assert dts.status_string(2) == "DTS_E_STATE"


def test_library_is_sm100a_cuda():
    from paper_2402_03106_b200 import dts
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", dts.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout, out.stdout + out.stderr


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "dts.h"\n'
                   'int main(){printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(dts_debug_in), sizeof(dts_debug_out),'
                   ' sizeof(dts_scene_desc), offsetof(dts_debug_out, E_next), offsetof(dts_debug_in, r),'
                   ' sizeof(dts_table_desc), offsetof(dts_scene_desc, parity_s_excess),'
                   ' offsetof(dts_scene_desc, tris), offsetof(dts_scene_desc, mats));}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    vals = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    from paper_2402_03106_b200 import dts
    mine = [dts.DEBUG_IN.itemsize, dts.DEBUG_OUT.itemsize, ctypes.sizeof(dts.SceneDesc),
            dts.DEBUG_OUT.fields["E_next"][1], dts.DEBUG_IN.fields["r"][1], ctypes.sizeof(dts.TableDesc),
            dts.SceneDesc.parity_s_excess.offset, dts.SceneDesc.tris.offset, dts.SceneDesc.mats.offset]
    assert vals == mine


def test_no_device_is_an_error_not_a_fallback():
    """Without a usable sm_100 device every entry point reports DTS_E_CUDA (or
    a validation error first) -- never a CPU result."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import dts_inputs as I
    from paper_2402_03106_b200 import dts
    with pytest.raises(dts.DtsError, match="DTS_E_CUDA"):
        dts.Scene(I.config(2))
    bad = I.config(2, g=1.5)
    with pytest.raises(dts.DtsError, match="DTS_E_INVALID_ARG"):
        dts.Scene(bad)


def test_product_package_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2402_03106_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower().replace("oracle/", ""), f


MESH_BAD = [
    ("no_materials", dict(n_mats=0), "n_mats"),
    ("material_index", dict(mat_index=5), "material index"),
    ("outside_box", dict(shift=(0.0, -0.05, 0.0)), "inside the box"),
    ("outside_sphere", dict(medium="sphere", radius=1.2), "inside the sphere"),
    ("degenerate", dict(degenerate=True), "degenerate"),
    ("rho", dict(mats=[(1.5, 0.0, 1.0)]), "rho, ks"),
]


@pytest.mark.parametrize("name,kw,msg", MESH_BAD, ids=[m[0] for m in MESH_BAD])
def test_mesh_validation_errors(name, kw, msg):
    """dts_scene_create rejects malformed meshes (include/dts.h) before it
    touches the device: DTS_E_INVALID_ARG with the reason."""
    import dts_inputs as I
    from paper_2402_03106_b200 import dts
    import numpy as np
    c = I.mesh_config()
    m = dict(c["mesh"])
    tris = np.array(m["tris"], dtype=np.float64).reshape(-1, 9)
    if "shift" in kw:
        tris = tris + np.tile(kw["shift"], 3)
    if kw.get("degenerate"):
        tris[0, 6:9] = tris[0, 3:6]
    mat = np.array(m["tri_mat"], dtype=np.int32)
    if "mat_index" in kw:
        mat[3] = kw["mat_index"]
    m.update(tris=tris, tri_mat=mat)
    if "mats" in kw:
        m["mats"] = kw["mats"]
    c["mesh"] = m
    for k in ("medium", "radius"):
        if k in kw:
            c[k] = kw[k]
            c["wall_mask"] = 0
    d = dts.scene_desc(c)
    if "n_mats" in kw:
        d.n_mats = kw["n_mats"]
    h = ctypes.c_void_p()
    st = dts._lib.dts_scene_create(ctypes.byref(d), ctypes.byref(h))
    assert dts._lib.dts_status_string(st).decode() == "DTS_E_INVALID_ARG"
    assert msg in dts._lib.dts_last_error().decode()
