"""CPU-side checks of the C ABI boundary: libplx.so loads without a GPU and
exports every entry point include/plx.h declares (no compute calls here)."""

import ctypes
import os
import re
import subprocess

from paper_2112_05131_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "plx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(plx_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (plx_\w+)", out))
    for name in declared_symbols():
        assert name in exported, name
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)
    assert lib.plx_version().decode().startswith("plx-b200")


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_scan_scratch_sizing_is_host_only():
    lib = _lib.load()
    assert lib.plx_scan_scratch_bytes(0) == 8
    assert lib.plx_scan_scratch_bytes(4096) == 16
    d = (ctypes.c_int64 * 3)(64, 64, 64)
    assert lib.plx_cell_occ_words(d) == 64 ** 3 // 32


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirrors in _lib.py have the C layout include/plx.h declares
    (sizeof and every field offset, checked by compiling the header)."""
    structs = {"plx_grid": _lib.PlxGrid, "plx_grad": _lib.PlxGrad,
               "plx_render_opts": _lib.PlxRenderOpts, "plx_rays": _lib.PlxRays,
               "plx_dp_peers": _lib.PlxDpPeers, "plx_step_args": _lib.PlxStepArgs,
               "plx_msi": _lib.PlxMsi, "plx_msi_grad": _lib.PlxMsiGrad,
               "plx_cameras": _lib.PlxCameras}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "plx.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True,
                                                       text=True, check=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)
