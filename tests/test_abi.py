"""C-ABI checks that need no GPU: libils.so loads, exports every symbol include/ils.h declares,
and the ctypes structs match the C layout (compiled with gcc against the header)."""
import os
import re
import shutil
import subprocess

import pytest

from paper_2203_15340_b200 import ils

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "ils.h")


def _declared():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"ILS_API\s+[\w\s\*]*?\b(ils_\w+)\s*\(", txt)))


def test_library_loads_and_exports_every_declared_symbol():
    if not os.path.exists(ils.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    lib = ils.load_library()
    names = _declared()
    assert len(names) >= 14
    for nm in names:
        assert hasattr(lib, nm), nm
    assert set(names) == set(ils.EXPORTED)
    out = subprocess.run(["nm", "-D", "--defined-only", ils.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (ils_\w+)", out))
    assert exported == set(names)


def test_host_only_entry_points():
    o = ils.ils_default_opts()
    assert o.stop == ils.ILS_STOP_XREF and o.inner_tol == 1e-12 and o.max_inner == 100000
    assert ils.load_library().ils_status_string(ils.ILS_ERR_NOT_SPD).decode().startswith("matrix not SPD")


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc missing")
def test_struct_layout_matches_header(tmp_path):
    src = tmp_path / "l.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "ils.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(ils_ext), sizeof(ils_opts),'
                   ' sizeof(ils_report), offsetof(ils_opts, seed), offsetof(ils_opts, x_hist),'
                   ' offsetof(ils_report, kernel_launches));return 0;}\n')
    exe = tmp_path / "l"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    import ctypes as C
    want = [C.sizeof(ils.IlsExt), C.sizeof(ils.IlsOpts), C.sizeof(ils.IlsReport),
            ils.IlsOpts.seed.offset, ils.IlsOpts.x_hist.offset, ils.IlsReport.kernel_launches.offset]
    assert got == want


def test_binding_rejects_wrong_dtypes_and_short_buffers():
    """The binding checks element types and lengths before handing pointers to the library (ADVICE
    round 1): float32 A / b, an int32 row pointer, a short b or a short x never reach libils."""
    import numpy as np
    A = np.ones((6, 3))
    with pytest.raises(TypeError):
        ils.ils_create(A.astype(np.float32), np.ones(6), 4, 2, 3)
    with pytest.raises(TypeError):
        ils.ils_create(A, np.ones(6, dtype=np.float32), 4, 2, 3)
    with pytest.raises(ValueError):
        ils.ils_create(A, np.ones(5), 4, 2, 3)
    with pytest.raises(ValueError):
        ils.ils_create(np.ones((5, 3)), np.ones(6), 4, 2, 3)
    vals = np.ones(6)
    with pytest.raises(TypeError):
        ils.ils_create(vals, np.ones(6), 4, 2, 3, row_ptr=np.arange(7, dtype=np.int32),
                       col_idx=np.zeros(6, dtype=np.int32))
    with pytest.raises(TypeError):
        ils.ils_create(vals, np.ones(6), 4, 2, 3, row_ptr=np.arange(7, dtype=np.int64),
                       col_idx=np.zeros(6, dtype=np.int64))
    ils._shape[12345] = (3, 1)
    import ctypes as C
    with pytest.raises(ValueError):
        ils.ils_sp_solve(C.c_void_p(12345), None, np.zeros(2), 0.0, 1)
    ils._shape.pop(12345)
