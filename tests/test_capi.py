"""The C-ABI library loads on CPU and exports every symbol the header declares."""

import ctypes
import os
import re

from paper_2510_08874_b200 import _capi

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "unimul_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"UM_API\s+(?:int|const char\*)\s+(um_\w+)\s*\(", text)))


def test_header_declares_the_bound_api():
    assert declared_symbols() == sorted(_capi.exported_symbols())


def test_library_exports_every_declared_symbol():
    lib = _capi.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value


def test_profiling_build_exports_the_same_api():
    """`make prof` (UM_GEMM_STALLS) builds the same C-ABI with profiling compiled in."""
    import pytest

    prof = os.path.join(os.path.dirname(_capi.LIB_PATH), "libunimul_b200_prof.so")
    if not os.path.exists(prof):
        pytest.skip("profiling build not present (make -C paper_2510_08874_b200/csrc prof)")
    lib = ctypes.CDLL(prof)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_version_and_errors_without_gpu():
    lib = _capi.load()
    assert b"sm_100a" in lib.um_version()
    n = ctypes.c_int64()
    rc = lib.um_iteration_offset(0, 0, 0, ctypes.byref(n))
    assert rc == _capi.UM_EVALUE and "nops" in _capi.last_error()
    gr, gc = ctypes.c_int64(), ctypes.c_int64()
    assert lib.um_most_square_grid(12, ctypes.byref(gr), ctypes.byref(gc)) == 0 and (gr.value, gc.value) == (3, 4)


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_capi.UmView) == 8 + 5 * 8 + 2 * 4
    assert ctypes.sizeof(_capi.UmMatDesc) == 6 * 8 + 2 * 4
    assert ctypes.sizeof(_capi.UmGemmOp) == 3 * ctypes.sizeof(_capi.UmView) + 48


def test_owner_rank_matches_python_tiling():
    from paper_2510_08874_b200 import tiling

    lib = _capi.load()
    for mapping, um in ((tiling.Mapping.BLOCK, _capi.UM_BLOCK), (tiling.Mapping.BLOCK_CYCLIC, _capi.UM_BLOCK_CYCLIC)):
        part = tiling.PartitionSpec(tiling.Shape2D(3, 2), tiling.Shape2D(2, 3), mapping)
        shape = tiling.Shape2D(17, 13)
        grid = tiling.grid_shape(part, shape)
        d = _capi.UmMatDesc(17, 13, 3, 2, 2, 3, um, 2)
        out = ctypes.c_int32()
        for t in grid.tiles():
            for rep in range(2):
                assert lib.um_owner_rank(ctypes.byref(d), 12, t.i, t.j, rep, ctypes.byref(out)) == 0
                assert out.value == tiling.owner_of(part, grid, t, 6) + 6 * rep


def test_struct_layouts_match_the_c_compiler(tmp_path):
    """sizeof / offsetof of every header struct, as gcc lays them out, equal the ctypes mirrors."""
    import shutil
    import subprocess

    import pytest

    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    structs = {"um_view": _capi.UmView, "um_mat_desc": _capi.UmMatDesc, "um_gemm_op": _capi.UmGemmOp,
               "um_get_desc": _capi.UmGetDesc, "um_exec_cfg": _capi.UmExecCfg, "um_exec_action": _capi.UmExecAction,
               "um_rank_plan": _capi.UmRankPlan, "um_reduce_step": _capi.UmReduceStep}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void) {"]
    for cname, cls in structs.items():
        lines.append(f'  printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'  printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("  return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-o", str(exe), str(src)], check=True)
    got = dict(ln.split() for ln in subprocess.run([str(exe)], capture_output=True, text=True,
                                                     check=True).stdout.splitlines())
    for cname, cls in structs.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, (cname, fname)


def test_execute_validates_without_gpu():
    lib = _capi.load()
    assert lib.um_execute(None, -1, None, 0, None) == _capi.UM_EVALUE
    bad = _capi.UmExecCfg(2, 0, 4, 4, 0, 0, 0, 0)               # prefetch_depth 0: runtime.py:35-37
    assert lib.um_execute(None, 0, None, 0, ctypes.byref(bad)) == _capi.UM_EVALUE
    assert "counts must be >= 1" in _capi.last_error()
