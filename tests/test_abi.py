"""The C-ABI library: builds, loads, exports exactly what the header declares,
and its argument struct matches the ctypes mirror.  No compute calls (CPU)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2601_04860_b200 import _native, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "divas_b200.h")


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _native.lib()


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(divas_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_exports():
    assert _declared() == sorted(_native.EXPORTS)


def test_library_exports_every_symbol(lib):
    nm = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH],
                        capture_output=True, text=True, check=True).stdout
    syms = {line.split()[-1] for line in nm.splitlines() if line.strip()}
    for name in _declared():
        assert name in syms, name
        assert getattr(lib, name) is not None


def test_version_and_error(lib):
    assert lib.divas_abi_version() == 11
    assert isinstance(lib.divas_last_error(), bytes)


def test_sm100a_code_only(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _c_layout(tmp_path, cname, fields):
    prog = tmp_path / f"layout_{cname}.c"
    body = "\n".join(f'printf("%zu\\n", offsetof({cname}, {f}));' for f in fields)
    prog.write_text(f"""
#include <stdio.h>
#include <stddef.h>
#include "divas_b200.h"
int main(void) {{ printf("%zu\\n", sizeof({cname})); {body} return 0; }}
""")
    exe = tmp_path / f"layout_{cname}"
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(prog), "-o", str(exe)], check=True)
    return [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                           check=True).stdout.split()]


@pytest.mark.parametrize("which", ["fuse", "trace", "record", "scene", "render_cfg", "copy2d"])
def test_struct_layout_matches_header(tmp_path, which):
    from paper_2601_04860_b200 import trace
    if which in ("scene", "render_cfg", "copy2d"):
        st, cname = {"scene": (_native.Scene, "divas_scene"),
                     "render_cfg": (_native.RenderCfg, "divas_render_cfg"),
                     "copy2d": (_native.Copy2D, "divas_copy2d")}[which]
        fields = [f[0] for f in st._fields_]
        vals = _c_layout(tmp_path, cname, fields)
        assert vals[0] == ctypes.sizeof(st)
        for f, off in zip(fields, vals[1:]):
            assert getattr(st, f).offset == off, f
        return
    if which == "record":
        names = list(trace.RECORD_DTYPE.names)
        vals = _c_layout(tmp_path, "divas_pair_record", names)
        assert vals[0] == trace.RECORD_DTYPE.itemsize
        for f, off in zip(names, vals[1:]):
            assert trace.RECORD_DTYPE.fields[f][1] == off, f
        return
    st, cname = ((_native.FuseArgs, "divas_fuse_args") if which == "fuse"
                 else (trace._TraceArgs, "divas_trace_args"))
    fields = [f[0] for f in st._fields_]
    vals = _c_layout(tmp_path, cname, fields)
    assert vals[0] == ctypes.sizeof(st)
    for f, off in zip(fields, vals[1:]):
        assert getattr(st, f).offset == off, f


def test_invalid_arguments_rejected_without_gpu(lib):
    """Argument validation happens before any CUDA call."""
    a = _native.FuseArgs()
    a.g = 0
    rc = lib.divas_fuse(ctypes.byref(a), None, 0, None)
    assert rc == 1
    assert b"grid" in lib.divas_last_error()
    assert lib.divas_refine(0, 1, 1, None, None, None, None, None, 0, None) == 1
    assert lib.divas_threshold(None, 10, 0.5, 0, None, None, None, None, 0, None) == 1


def test_render_arguments_rejected_without_gpu(lib):
    """Scene / config validation of the fixture producers (RenderConfig's own
    checks, render.py:44-50) happens before any CUDA call."""
    sc = _native.Scene()
    sc.n_prims = _native.MAX_PRIMS + 1
    cfg = _native.RenderCfg(16, 0.5, 6.0, 0.75, 1e-4)
    assert lib.divas_render(ctypes.byref(sc), ctypes.byref(cfg), 1, None, 4, 4, *([None] * 7),
                            None) == 1
    assert b"primitives" in lib.divas_last_error()
    sc.n_prims = 0
    for bad in ((0, 0.5, 6.0, 0.75), (16, 6.0, 0.5, 0.75), (16, 0.5, 6.0, 0.0),
                (16, 0.5, 6.0, 1.5)):
        cfg = _native.RenderCfg(*bad, 1e-4)
        assert lib.divas_render(ctypes.byref(sc), ctypes.byref(cfg), 1, None, 4, 4,
                                *([None] * 7), None) == 1
        assert lib.divas_march_rays(ctypes.byref(sc), ctypes.byref(cfg), 1, None, None, None,
                                    None, None) == 1
    o = (ctypes.c_double * 3)()
    assert lib.divas_bake_density(ctypes.byref(sc), 0, o, 0.1, 0, o, o, None, None) == 1
