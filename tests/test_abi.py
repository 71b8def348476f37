"""The C-ABI library loads without a GPU and exports every symbol include/pf.h declares;
host-side validation (topology / model) works without a device."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1812_01502_b200 import inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pfb():
    from paper_1812_01502_b200 import build, pf
    build.build()
    return pf


def _declared():
    src = open(os.path.join(ROOT, "include", "pf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(pfb):
    names = _declared()
    assert "pf_init" in names and "pf_step" in names and "pf_estimate" in names
    L = pfb.lib()
    for n in names:
        assert hasattr(L, n), n
    assert sorted(pfb.EXPORTED) == names


@pytest.mark.parametrize("N,M,ok", [(1024, 64, True), (1 << 28, 64, True), (64, 64, False), (96, 32, False),
                                    (1024, 1, False), (1024, 3, False), (1 << 14, 4096, True), (1 << 14, 8192, False), (1 << 14, 16384, False),
                                    (4, 2, True), (1 << 31, 64, False)])
def test_topology_validation(pfb, N, M, ok):
    p = inputs.model_params(inputs.CONFIGS["C4"])
    nbytes = pfb.pf_workspace_bytes(p, N, M)
    assert (nbytes > 0) == ok


def test_model_validation(pfb):
    p = dict(inputs.model_params(inputs.CONFIGS["C4"]))
    assert pfb.pf_workspace_bytes(p, 1 << 16, 64) > 0
    bad = dict(p)
    LQ = p["LQ"].copy()
    LQ[0, 1] = 1.0  # not lower triangular
    bad["LQ"] = LQ
    assert pfb.pf_workspace_bytes(bad, 1 << 16, 64) == 0
    bad = dict(p)
    bad["d"] = 3
    assert pfb.pf_workspace_bytes(bad, 1 << 16, 64) == 0
    sv = inputs.model_params(inputs.CONFIGS["C3"])
    assert pfb.pf_workspace_bytes(sv, 1 << 16, 32) > 0
    assert pfb.pf_workspace_bytes(sv, 1 << 26, 8192) > 0  # C5's largest group (d = 1)


def test_workspace_scales(pfb):
    p = inputs.model_params(inputs.CONFIGS["C4"])
    a = pfb.pf_workspace_bytes(p, 1 << 20, 64)
    b = pfb.pf_workspace_bytes(p, 1 << 21, 64)
    assert 1.9 < b / a < 2.1
    dbg = pfb.pf_workspace_bytes(p, 1 << 20, 64, pfb.PF_FLAG_DEBUG)
    assert dbg > a + (1 << 20) * 14 * 4


def test_scheme_flags_reserve_their_buffers(pfb):
    """PF_FLAG_ADAPTIVE / _AIRPF / _MULTINOMIAL add the buffers include/pf.h states."""
    p = inputs.model_params(inputs.CONFIGS["C4"])
    N, M = 1 << 20, 64
    base = pfb.pf_workspace_bytes(p, N, M)
    ad = pfb.pf_workspace_bytes(p, N, M, pfb.PF_FLAG_ADAPTIVE)
    air = pfb.pf_workspace_bytes(p, N, M, pfb.PF_FLAG_AIRPF)
    mn = pfb.pf_workspace_bytes(p, N, M, pfb.PF_FLAG_MULTINOMIAL)
    assert ad - base >= 8 * N            # two fp32 log-weight buffers
    assert air - base >= 12 * (N // M)   # island map (int32) + island log-means (fp64)
    assert mn - base >= 8 * N            # log-weights + tile CDFs (fp32)
    both = pfb.pf_workspace_bytes(p, N, M, pfb.PF_FLAG_ADAPTIVE | pfb.PF_FLAG_MULTINOMIAL)
    assert both >= max(ad, mn)


def test_guard_flag_adds_gaps(pfb):
    """PF_FLAG_GUARD: one PF_GUARD_BYTES gap after every workspace region, whatever the
    other flags (the region count is fixed by the layout)."""
    p = inputs.model_params(inputs.CONFIGS["C4"])
    N, M = 1 << 20, 64
    for flags in (0, pfb.PF_FLAG_DEBUG, pfb.PF_FLAG_ADAPTIVE | pfb.PF_FLAG_AIRPF | pfb.PF_FLAG_MULTINOMIAL):
        plain = pfb.pf_workspace_bytes(p, N, M, flags)
        guarded = pfb.pf_workspace_bytes(p, N, M, flags | pfb.PF_FLAG_GUARD)
        extra = guarded - plain
        assert extra > 0 and (extra - 256) % 4096 == 0  # gaps + the 256-byte counter region
        assert 30 <= (extra - 256) // 4096 <= 60  # one gap per region (+ the guard counter's own)
