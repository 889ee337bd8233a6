"""The C-ABI library loads without a GPU and exports every function the
headers in include/ declare; the ctypes mirror has the C struct layouts."""
import ctypes as C
import re
import subprocess
import textwrap
from pathlib import Path

import pytest

from paper_2106_14189_b200 import _abi as A

ROOT = Path(__file__).resolve().parents[1]
HEADERS = [ROOT / "include" / "djg.h", ROOT / "include" / "djg_host.h"]


def declared_functions():
    names = set()
    for h in HEADERS:
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        for m in re.finditer(r"^[A-Za-z_][\w \*]*?\b(djg_\w+)\s*\(", text, flags=re.M):
            names.add(m.group(1))
    return names


def test_headers_declare_the_mirrored_exports():
    declared = declared_functions()
    mirrored = {name for name, _, _ in A.EXPORTS}
    assert declared == mirrored, (declared - mirrored, mirrored - declared)


def test_library_loads_and_exports_all_symbols():
    lib = A.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(A.LIB_PATH)], capture_output=True, text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_status_strings_without_gpu():
    lib = A.load_library()
    assert lib.djg_status_string(A.DJG_E_INVERSION) == b"element inversion"
    assert lib.djg_status_string(A.DJG_E_DIVERGENCE) == b"divergence"


def test_create_rejects_bad_descriptor_without_gpu():
    lib = A.load_library()
    d = A.djg_desc()
    d.precision = 3
    h = C.c_void_p()
    assert lib.djg_create(C.byref(d), C.byref(h)) == A.DJG_E_CONFIG
    assert h.value is None


STRUCTS = ["djg_material_params", "djg_scenario_spec", "djg_image_ptrs", "djg_image_scalars", "djg_report",
           "djg_assemble_stats", "djg_desc", "djg_engine_info", "djg_mesh_desc", "djg_step_desc", "djg_partition_info"]


def test_struct_layouts_match_c(tmp_path):
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "djg_host.h"', "int main(void){"]
    for s in STRUCTS:
        cls = getattr(A, s)
        lines.append(f'printf("{s} %zu\\n", sizeof({s}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{s}.{f} %zu\\n", offsetof({s}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-std=c11", f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    for s in STRUCTS:
        cls = getattr(A, s)
        assert int(got[s]) == C.sizeof(cls), s
        for f, _ in cls._fields_:
            assert int(got[f"{s}.{f}"]) == getattr(cls, f).offset, (s, f)
