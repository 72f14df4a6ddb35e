"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every
symbol include/smallkv.h declares, and its pure-host logic is right."""
from __future__ import annotations

import ctypes
import json
import os
import re

import pytest

from paper_2508_02751_b200 import build as kbuild
from paper_2508_02751_b200 import smallkv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))


@pytest.fixture(scope="module")
def lib():
    kbuild.build()
    return smallkv.load()


def test_header_symbols_exported(lib):
    src = open(os.path.join(ROOT, "include", "smallkv.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\**\s+\**(smallkv_[a-z_0-9]+)\(",
                              src, re.M))
    assert declared == set(smallkv.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def test_version(lib):
    assert "sm_100a" in smallkv.version()


def test_budget_from_tau_paper_example(lib):
    g = GOLDEN["budget_tau"]
    assert list(smallkv.budget_from_tau(g["tau"], g["n"])) == g["expect"]


@pytest.mark.parametrize("tau,n", [(0.2, 4096), (0.05, 32768), (0.5, 32768), (0.35, 200),
                                   (1.0, 7), (0.2, 0)])
def test_budget_from_tau_half_cost_invariant(lib, tau, n):
    """K + R + M/2 <= tau n (marginal tokens cost half), 2:1:2 ratio."""
    K, R, M = smallkv.budget_from_tau(tau, n)
    assert K + R + M / 2 <= tau * n + 1e-9
    assert K == M and abs(K - 2 * R) <= 1
    assert K + R + M <= n


def test_budget_from_tau_rejects(lib):
    with pytest.raises(smallkv.SmallKVError):
        smallkv.budget_from_tau(0.0, 10)
    with pytest.raises(smallkv.SmallKVError):
        smallkv.budget_from_tau(1.5, 10)


def test_validation_errors_before_launch(lib):
    """Host checks return non-OK without touching a device."""
    c = smallkv.CCache(0, 0, 0, 1, 1, 64, 1, 4, 2, 64)
    b = smallkv.CBatch(0, 1, 16)
    assert lib.smallkv_select_workspace_size(ctypes.byref(c), ctypes.byref(b), 4) > 0
    rc = lib.smallkv_attend(0, 0, None, ctypes.byref(c), ctypes.byref(b), None, 1, 2, None,
                            None, None, None, None, None, None, 0, None, 0, None)
    assert rc == 1  # ERR_NULL
    assert b"NULL" in lib.smallkv_last_error()
    bad = smallkv.CCache(16, 16, 16, 1, 1, 64, 1, 4, 2, 96)  # head_dim 96
    rc = lib.smallkv_select(16, ctypes.byref(bad), ctypes.byref(b), 16, 4, None, None, None,
                            None, None, None, None, None, None, 0, None, None)
    assert rc == 2  # ERR_SHAPE
    rc = lib.smallkv_match_heads(16, 1, 16, 1, 600, 3, 16, 16, 16, 1 << 20, None)
    assert rc == 2  # window > 512


def test_kv_bytes_model():
    """Eq. 7 byte model vs SPEC's worked value and P:628's ratio."""
    from paper_2508_02751_b200 import bytes_model as bm
    g = GOLDEN["hot_bytes_qwen2_7b"]
    assert bm.kv_cache_bytes(g["L"], g["N_kv"], g["D_kv"], g["S"], g["B"], g["C_b"]) == g["bytes"]
    r = bm.kv_cache_bytes(80, 8, 128, 1, 1, 2) / bm.kv_cache_bytes(28, 4, 128, 1, 1, 2)
    assert abs(r - GOLDEN["kv_ratio_72b_7b"]["value"]) < GOLDEN["kv_ratio_72b_7b"]["tol"]


def test_f3_match_window_host():
    """smallkv_match_window (host) = SPEC's window decisions (R17)."""
    w = GOLDEN["matching_window"]
    for n, want in w["cases"]:
        got = smallkv.match_window(n, w["min_len"], w["max_len"], keep_last=True)
        assert (None if got is None else [got[0], got[0] + got[1]]) == want
    assert smallkv.match_window(1000, keep_last=False) == (0, 200)
    with pytest.raises(smallkv.SmallKVError):
        smallkv.match_window(10, 200, 100)


def test_next_row_entry_points_validate_before_launch(lib):
    """f2 / f3 / f4 entry points: argument errors are reported on the host
    (no device needed), with the documented status codes."""
    P = ctypes.c_void_p
    c = smallkv.CCache(16, 16, 16, 4, 4, 16, 2, 8, 2, 128)
    b = smallkv.CBatch(16, 2, 64)
    bu = smallkv.CBudgets(16, 16, 16, 8, 8)
    # f2: G = 8 / 2 = 4 ok; H % H_kv != 0 rejected
    rc = lib.smallkv_select_group(16, ctypes.byref(c), ctypes.byref(b), 16, 2, 8, 3,
                                  ctypes.byref(bu), 16, 16, 16, 16, 16, 16, 16, 16, 1 << 20, None)
    assert rc == 2 and b"invalid" in lib.smallkv_last_error()
    rc = lib.smallkv_select_group(16, ctypes.byref(c), ctypes.byref(b), 16, 2, 8, 2,
                                  ctypes.byref(bu), 16, 16, None, 16, 16, 16, 16, 16, 1 << 20, None)
    assert rc == 1
    # f3: window length bounds
    rc = lib.smallkv_prefill_scores(16, ctypes.byref(c), 0, 0, 2000, 16, None)
    assert rc == 2
    rc = lib.smallkv_prefill_scores(None, ctypes.byref(c), 0, 0, 10, 16, None)
    assert rc == 1
    # f4: capacity must be a multiple of 4; state size reported
    assert lib.smallkv_tier_state_size(ctypes.byref(c), ctypes.byref(b), 2, 30) == 0
    assert lib.smallkv_tier_state_size(ctypes.byref(c), ctypes.byref(b), 2, 32) > 0
    rc = lib.smallkv_tier_init(16, 8, ctypes.byref(c), ctypes.byref(b), 2, 32, None)
    assert rc == 4   # ERR_WORKSPACE: state too small
    rc = lib.smallkv_tier_update(0, 3, ctypes.byref(c), 16, 16, 32, ctypes.byref(b), 16, 2, 16,
                                 ctypes.byref(bu), 16, 16, 16, 16, 0, 16, 1 << 30, None)
    assert rc == 2   # layers [0, 3) past the 2 LLM layers
