"""The C-ABI library loads on a GPU-less host and exports every symbol include/dd_api.h declares.
No compute calls (no GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dd_api.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dd_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_four_calls():
    names = _declared()
    for n in ("dd_setup", "dd_apply_schur", "dd_apply_precond", "dd_pcg_solve"):
        assert n in names


def test_library_exports_every_declared_symbol():
    import __graft_entry__ as ge
    ge.build()
    from paper_2211_15308_b200 import binding
    lib = ctypes.CDLL(binding.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(binding.EXPORTS) == set(_declared())


def test_setup_validation_without_gpu():
    # argument validation happens before any CUDA call
    from paper_2211_15308_b200 import binding
    lib = binding.load()
    mesh = binding._Mesh(4, 8, 0)
    h = ctypes.c_void_p()
    import numpy as np
    K = np.ones(1); mu = np.ones(1); c0 = np.zeros(1)
    st = lib.dd_setup(ctypes.byref(mesh), 1, K.ctypes.data, mu.ctypes.data, 0, None, None, c0.ctypes.data, 1, 0,
                      None, None, ctypes.byref(h))
    assert st == binding.DD_EINVAL and b"dim" in lib.dd_last_error()
    mesh = binding._Mesh(2, 8, 0)
    Kb = np.array([-1.0])
    st = lib.dd_setup(ctypes.byref(mesh), 1, Kb.ctypes.data, mu.ctypes.data, 0, None, None, c0.ctypes.data, 1, 0,
                      None, None, ctypes.byref(h))
    assert st == binding.DD_EINVAL
    poles = np.array([0.1]); res = np.ones(1)
    st = lib.dd_setup(ctypes.byref(mesh), 1, K.ctypes.data, mu.ctypes.data, 1, poles.ctypes.data, res.ctypes.data,
                      c0.ctypes.data, 1, 0, None, None, ctypes.byref(h))
    assert st == binding.DD_EINVAL and b"pole" in lib.dd_last_error()
    assert lib.dd_interface_size(None) == -1


def test_bench_live_columns():
    """bench.py's algorithmic-work count under live-tile compaction (host logic): the apply at
    iteration k multiplies only the tiles holding a column with iters >= k, once the batch has at
    least 6 tiles of 64 columns (the library's threshold); otherwise every column every time."""
    import bench
    its = np.array([3] * 64 + [5] * 64 + [2] * 300)            # 7 tiles of 64 (last ragged)
    assert bench.live_columns(its, True) == [428, 428, 128, 64, 64]
    assert bench.live_columns(its, False) == [428] * 5
    its32 = np.repeat([4, 2, 3, 1, 4, 4, 2, 1, 1, 1, 1, 1], 32)  # 384 columns: 6 tiles of 64
    lc = bench.live_columns(its32, True, bn=32)
    assert lc == [384, 32 * 6, 32 * 4, 32 * 3]
    assert bench.live_columns(np.array([3] * 256), True, bn=32) == [256] * 3   # 4 tiles of 64: off
