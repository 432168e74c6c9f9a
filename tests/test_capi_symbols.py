"""CPU-side checks of the boundary: the shared library builds for sm_100a, loads
without a GPU, and exports every entry point include/dmm.h declares."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "dmm.h")) as f:
        return re.findall(r"DMM_API\s+[\w\s\*]+?\b(dmm_\w+)\s*\(", f.read())


@pytest.fixture(scope="module")
def lib():
    from paper_1601_06274_b200 import _build
    path = _build.build()
    return ctypes.CDLL(path)


def test_header_declares_entry_points():
    names = _declared()
    assert "dmm_solve" in names and "dmm_cost_volume" in names and "dmm_result" in names
    import paper_1601_06274_b200 as dmm
    assert sorted(names) == sorted(dmm.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name


def test_only_api_symbols_exported(lib):
    from paper_1601_06274_b200 import _build
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True, text=True).stdout
    text_syms = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert text_syms == set(_declared())


def test_sm100a_cubin_present():
    from paper_1601_06274_b200 import _build
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_only_calls_without_gpu(lib):
    """Workspace sizing and argument checks need no device."""
    import paper_1601_06274_b200 as dmm
    L = dmm.load_library()
    cfg = dmm.DmmConfig(1242, 375, 0, 127, 2, 3, 3, 4, 4, -1, 1, 4)
    n = L.dmm_workspace_bytes(ctypes.byref(cfg))
    px, cells = 1242 * 375, 1242 * 375 * 128
    rec = 2 * 128 + 16                 # compact u16-span dual record per pixel
    assert n >= cells * (1 + 2 * 4) + 2 * px * rec + px * 11
    bad = dmm.DmmConfig(1242, 375, 0, 300, 2, 3, 3, 4, 4, -1, 1, 4)   # K > 256
    assert L.dmm_workspace_bytes(ctypes.byref(bad)) == 0
    h = ctypes.c_void_p()
    assert L.dmm_create(ctypes.byref(bad), None, 0, 0, ctypes.byref(h)) == 1   # DMM_E_ARG
    assert L.dmm_status_str(3) == b"invalid state"
    # span bound (2*w*min(T,K-1) + maxD) * 2^F > 65535 -> DMM_E_RANGE (6)
    big = dmm.DmmConfig(64, 32, 0, 63, 2, 255, 255, 63, 8, -1, 1, 4)
    assert L.dmm_create(ctypes.byref(big), ctypes.c_void_p(256), 1 << 40, 0, ctypes.byref(h)) == 6
    assert L.dmm_launch_count(None) == 0


def test_no_cpu_fallback_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1601_06274_b200 as dmm
    with pytest.raises(dmm.DmmError):
        dmm.Context(width=8, height=8, d_min=0, d_max=7)


def test_product_path_does_not_import_oracle():
    src_dir = os.path.join(ROOT, "paper_1601_06274_b200")
    for dp, _, fns in os.walk(src_dir):
        for fn in fns:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                with open(os.path.join(dp, fn)) as f:
                    txt = f.read()
                assert "import oracle" not in txt and "from oracle" not in txt and "dmm_oracle" not in txt, fn
