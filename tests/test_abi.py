"""The C-ABI library loads and exports every symbol include/husky.h declares
(no compute calls: this runs without a GPU), plus the host-only entry points."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "husky.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(husky_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_the_north_star_entry_points():
    names = _declared()
    for must in ("husky_encode", "husky_sort", "husky_sort_multi"):
        assert must in names


def test_library_exports_every_declared_symbol():
    import paper_2012_00866_b200 as h
    lib = ctypes.CDLL(h.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_declared()) == set(h.EXPORTED)


def test_library_is_sm100a_only():
    import subprocess
    import paper_2012_00866_b200 as h
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", h.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_unit_bytes_and_workspace_queries():
    import paper_2012_00866_b200 as h
    assert h.husky_unit_bytes(0) == 1 and h.husky_unit_bytes(1) == 2 and h.husky_unit_bytes(7) == 0
    assert h.husky_unit_bytes(2) == 1 and h.husky_unit_bytes(3) == 1
    assert h.husky_sort_keys_workspace(2, 1000) > 1000 * 20
    with pytest.raises(h.HuskyError):
        h.husky_sort_keys_workspace(3, 10)
    w1 = h.husky_sort_workspace(0, 10_000_000)
    w2 = h.husky_sort_workspace(0, 20_000_000)
    assert 10_000_000 * 20 < w1 < w2
    with pytest.raises(h.HuskyError) as e:
        h.husky_sort_workspace(5, 10)
    assert e.value.status == 1 and "coder" in h.husky_last_error()


def test_host_many_workspace_slots():
    """husky_sort_host_many: `depth` input slots (device inputs + sort workspace)
    and depth + 1 output slots (perm, sorted units, sorted offsets) -- each added
    input slot costs at least one sort workspace, each added output slot at
    least the outputs' bytes."""
    import paper_2012_00866_b200 as h
    n, u = 1_000_000, 16_000_000
    sort_ws = h.husky_sort_workspace(0, n, u)
    outs = n * 4 + u + (n + 1) * 8
    w1, w2, w3 = (h.husky_sort_host_many_workspace(0, n, u, d) for d in (1, 2, 3))
    assert w1 >= sort_ws + u + (n + 1) * 8 + 2 * outs
    assert w2 - w1 == w3 - w2 >= sort_ws + u + (n + 1) * 8 + outs
    with pytest.raises(h.HuskyError):
        h.husky_sort_host_many_workspace(0, n, u, 0)


def test_select_splitters_host():
    """The sample sort's splitter rule (host copy, no GPU): sample strings sorted
    in the sort order (ties by index), positions floor(k*m/P)."""
    import paper_2012_00866_b200 as h
    import workloads as W
    rng = np.random.default_rng(0)
    strings = [rng.integers(0x61, 0x64, size=int(rng.integers(0, 6))).tolist() for _ in range(4 * 4096)]
    w = W.from_strings(strings, 0)
    idx = h.husky_select_splitters(0, w.units, w.offsets, 4)
    order = sorted(range(len(strings)), key=lambda i: (strings[i], i))
    m = len(strings)
    assert idx.tolist() == [order[k * m // 4] for k in (1, 2, 3)]
    assert h.husky_select_splitters(0, w.units, w.offsets, 1).size == 0
    u = W.from_strings([[0x4E00, 5], [0x4E00], [3]], 1)
    assert h.husky_select_splitters(1, u.units, u.offsets, 3).tolist() == [1, 0]
