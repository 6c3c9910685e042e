"""C-ABI library: loads on CPU, exports every symbol include/ffst.h declares, and
its host-only planner logic (index order, pruning ranges, Nyquist planes)
agrees with the oracle.  No device calls (CPU only)."""
import re
from pathlib import Path

import numpy as np
import pytest

import oracle as O

F = pytest.importorskip("paper_1202_1773_b200")
ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_header_symbols():
    header = (ROOT / "include" / "ffst.h").read_text()
    declared = set(re.findall(r"^\s*(?:ffst_status|int|const char\*)\s+(ffst_[a-z0-9_]+)\s*\(", header, re.M))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(F.lib, name), name
    assert declared == set(F.EXPORTED)


def test_scales_and_counts_match_oracle():
    for n in (4, 5, 15, 16, 63, 64, 255, 256, 1023, 1024, 4096):
        assert F.scales_for_size(n) == O.scales_for_size(n)
    for j0 in range(1, 9):
        assert F.num_shearlets(j0) == O.num_shearlets(j0)
    with pytest.raises(F.FFSTError):
        F.scales_for_size(3)


@pytest.mark.parametrize("j0", [1, 2, 3, 4, 5, 6])
def test_index_table_matches_oracle(j0):
    for i in range(O.num_shearlets(j0)):
        assert F.index_to_params(j0, i) == O.index_to_params(j0, i + 1)
        assert F.params_to_index(j0, *F.index_to_params(j0, i)) == i
    with pytest.raises(F.FFSTError):
        F.index_to_params(j0, O.num_shearlets(j0))
    with pytest.raises(F.FFSTError):
        F.params_to_index(j0, 3, 0, 0)


def _uncropped(n, i):
    """Oracle spectrum on the odd (n+1) grid before the even-n crop."""
    j0 = O.scales_for_size(n)
    axis, *_ = O.frequency_grid(n, j0)
    w1, w2 = np.meshgrid(axis, axis)
    kind, j, k = O.index_to_params(j0, i + 1)
    return O.ffst_oracle._spectrum_on_grid(w1, w2, kind, j, k)


@pytest.mark.parametrize("n", [4, 8, 16, 32, 64, 128, 256, 33, 48, 65, 100])
def test_pruning_range_is_a_superset(n):
    # the kernels evaluate sym(psi) only on columns |u1| in [lo, hi]; the oracle's
    # (uncropped) spectrum must vanish on every other column.
    j0 = O.scales_for_size(n)
    h = n // 2
    for i in range(O.num_shearlets(j0)):
        s = _uncropped(n, i)                      # columns index u1 = -h..h
        cols = np.nonzero(np.any(s != 0.0, axis=0))[0] - h
        lo, hi = F.plane_support(n, i)
        assert 0 <= lo <= hi <= h
        assert np.all(np.abs(cols) >= lo) and np.all(np.abs(cols) <= hi), (n, i, lo, hi)


@pytest.mark.parametrize("n", [4, 8, 16, 32, 64, 128, 33, 48, 65, 100])
def test_nyquist_classification(n):
    # a plane has an anti-symmetric part on the even grid iff psi(u1,-n/2) != psi(u1,+n/2) or
    # psi(-n/2,u2) != psi(+n/2,u2) somewhere.
    # odd n: the grid has no -n/2 bin: no plane has a Nyquist part
    j0 = O.scales_for_size(n)
    for i in range(O.num_shearlets(j0)):
        if n % 2:
            assert not F.plane_is_nyquist(n, i)
            continue
        s = _uncropped(n, i)
        differs = (np.max(np.abs(s[0, :] - s[-1, :])) > 1e-12) or (np.max(np.abs(s[:, 0] - s[:, -1])) > 1e-12)
        assert F.plane_is_nyquist(n, i) == differs, (n, i)


def test_invalid_sizes_rejected():
    with pytest.raises(F.FFSTError):
        F.plane_support(3, 0)
    with pytest.raises(F.FFSTError):
        F.shard_planes(64, 30, 0)        # more shards than the 29 planes
    with pytest.raises(F.FFSTError):
        F.plane_support(64, 29)
