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
    assert dts.abi_version() == 1
    assert dts.status_string(2) == "DTS_E_STATE"


def test_library_is_sm100a_cuda():
    from paper_2402_03106_b200 import dts
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", dts.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout, out.stdout + out.stderr


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "dts.h"\n'
                   'int main(){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(dts_debug_in), sizeof(dts_debug_out),'
                   ' sizeof(dts_scene_desc), offsetof(dts_debug_out, E_next), offsetof(dts_debug_in, r),'
                   ' sizeof(dts_table_desc), offsetof(dts_scene_desc, parity_s_excess));}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    vals = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    from paper_2402_03106_b200 import dts
    mine = [dts.DEBUG_IN.itemsize, dts.DEBUG_OUT.itemsize, ctypes.sizeof(dts.SceneDesc),
            dts.DEBUG_OUT.fields["E_next"][1], dts.DEBUG_IN.fields["r"][1], ctypes.sizeof(dts.TableDesc),
            dts.SceneDesc.parity_s_excess.offset]
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
