"""CPU-side checks of the drop-in boundary: the C-ABI library builds, loads,
and exports every entry point include/owb200.h declares (no compute calls —
there is no GPU here), and the ctypes structs match the C layout."""

import ctypes
import os
import re
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "owb200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|int64_t)\s+(ow_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2502_16310_b200 import _build

    return _build.build()


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("ow_fill_bins_count", "ow_fill_bins_emit", "ow_mark_near_wall", "ow_propagate_marks",
                 "ow_refine_marked", "ow_cell_face_links_count", "ow_lattice_links_count", "ow_stl_binary_to_soa"):
        assert must in names


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.ow_version() == 10000


def test_library_is_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("src", ["ow_nearwall.cu", "ow_lattice.cu", "ow_binning.cu"])
def test_no_fma_contraction_in_ptx(src, tmp_path):
    """-fmad=false must hold: no fused multiply-add in the emitted PTX (the
    FFMAs in SASS belong to ptxas's IEEE div.rn/sqrt.rn expansions only)."""
    from paper_2502_16310_b200 import _build

    out = tmp_path / "k.ptx"
    flags = [f for f in _build.NVCC_FLAGS if f not in ("-shared", "-lineinfo")]
    flags = [f.replace("code=sm_100a", "code=compute_100a") for f in flags]
    subprocess.run([_build.nvcc(), *flags, "-ptx", "-I", os.path.join(REPO, "include"), "-o", str(out),
                    os.path.join(_build.CSRC, src)], check=True, capture_output=True)
    ptx = out.read_text()
    assert "fma.rn.f32" not in ptx and "fma.rn.f64" not in ptx
    assert "mul.rn.f32" in ptx or "mul.f32" in ptx


def test_struct_layouts_match_c():
    from paper_2502_16310_b200 import _lib

    src = r'''
    #include <stdio.h>
    #include <stddef.h>
    #include "owb200.h"
    int main(){printf("%zu %zu %zu %zu %zu\n", sizeof(ow_forest), sizeof(ow_grid), sizeof(ow_face_summary),
                       offsetof(ow_forest, d_level), offsetof(ow_forest, grow));}
    '''
    exe = "/tmp/ow_layout"
    subprocess.run(["g++", "-x", "c++", "-I", os.path.join(REPO, "include"), "-", "-o", exe], input=src,
                   text=True, check=True)
    vals = [int(x) for x in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    assert vals == [ctypes.sizeof(_lib.ForestView), ctypes.sizeof(_lib.Grid), ctypes.sizeof(_lib.FaceSummary),
                    _lib.ForestView.d_level.offset, _lib.ForestView.grow.offset]


def test_no_gpu_means_loud_failure():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2502_16310_b200 as ow

    with pytest.raises(ow.OctowallError, match="CUDA device"):
        ow.init_root_grid(ow.Aabb((0, 0), (1, 1)), (4, 4))


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of the C structs have the C compiler's sizes/offsets."""
    import ctypes as C
    import shutil
    import subprocess

    from paper_2502_16310_b200 import _lib

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    src = tmp_path / "sz.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "owb200.h"\n'
        "int main(){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(ow_grid), sizeof(ow_forest),"
        " sizeof(ow_face_summary), sizeof(ow_nearwall_params), sizeof(ow_nearwall_result), sizeof(ow_g2g_params),"
        " sizeof(ow_g2g_result), offsetof(ow_g2g_result, nw)); return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.run([cc, "-I", os.path.join(REPO, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [C.sizeof(_lib.Grid), C.sizeof(_lib.ForestView), C.sizeof(_lib.FaceSummary),
            C.sizeof(_lib.NearWallParamsC), C.sizeof(_lib.NearWallResultC), C.sizeof(_lib.G2GParamsC),
            C.sizeof(_lib.G2GResultC), _lib.G2GResultC.nw.offset]
    assert got == want


def test_cpulist_parser():
    """sysfs cpulist syntax used by bind_host_numa (pinned buffers on the GPU's node)."""
    from paper_2502_16310_b200 import _lib

    assert _lib._cpulist("0-3,8,10-11\n") == {0, 1, 2, 3, 8, 10, 11}
    assert _lib._cpulist("5") == {5}
    assert _lib._cpulist("") == set()
