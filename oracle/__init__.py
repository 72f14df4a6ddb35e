"""TEST INFRASTRUCTURE ONLY — the fp64 CPU oracle of SmallKV's decode hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2508_02751_b200``) never imports it and has no CPU fallback.

The arithmetic lives in ``smallkv_oracle.c`` (plain C, fp64, one function per
step of the paper, each citing its passage); this module only builds it with
gcc and marshals numpy arrays through ctypes.  It shares no code with the CUDA
path.  Parity pins: ``tests/test_oracle_pins.py``.

Functions whose parity is pinned: all of them; the choice
among the readings R1/R2/R9 is documented, not pinned (no printed worked
example of Eq. 6 exists) — "parity unpinned" for those readings only.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "smallkv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc -O2 -fopenmp (fp64, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
               "-fno-fast-math", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


class _Cache(ctypes.Structure):
    _fields_ = [("k", ctypes.c_void_p), ("v", ctypes.c_void_p),
                ("block_table", ctypes.c_void_p), ("num_pages", ctypes.c_int64),
                ("max_blocks", ctypes.c_int32), ("page_size", ctypes.c_int32),
                ("num_layers", ctypes.c_int32), ("num_q_heads", ctypes.c_int32),
                ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32)]


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            i32 = ctypes.c_int32
            lib.oracle_slm_row.argtypes = [P, P, i32, i32, i32, i32, P, P, P, P]
            lib.oracle_split.argtypes = [P, i32, i32, i32, i32, P, P, P]
            lib.oracle_select.argtypes = [P, P, P, i32, i32, P, i32, P, P, P, i32, i32,
                                          P, P, P, P, P, P]
            lib.oracle_select_acc.argtypes = [P, P, P, i32, i32, P, i32, P, P, P, i32, i32,
                                              P, P, P, P, P, P, P]
            lib.oracle_attend.argtypes = [i32, i32, P, P, P, i32, P, P, P, i32, P, P, P,
                                          i32, i32, P, P]
            lib.oracle_select_group.argtypes = [i32, i32, i32, P, P, P, i32, P, i32, P, P, P,
                                                i32, i32, P, P, P, P]
            lib.oracle_attend_group.argtypes = lib.oracle_attend.argtypes
            lib.oracle_match_window.argtypes = [i32, i32, i32, i32, P, P]
            lib.oracle_match_window.restype = ctypes.c_int
            lib.oracle_prefill_scores.argtypes = [P, P, i32, i32, i32, P]
            lib.oracle_topk.argtypes = [P, i32, i32, P]
            lib.oracle_match_heads.argtypes = [P, i32, P, i32, i32, i32, P, P]
            lib.oracle_accumulate_scores.argtypes = [P, i32, P]
            lib.oracle_num_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _c(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=dtype)


def _bf16_bits(t) -> np.ndarray:
    """torch bf16 tensor (any device) or uint16 array -> contiguous uint16 numpy."""
    if isinstance(t, np.ndarray):
        return _c(t, np.uint16)
    import torch  # local: the oracle itself does not need torch
    return t.detach().contiguous().cpu().view(torch.int16).numpy().view(np.uint16)


def _i32(t) -> np.ndarray:
    if isinstance(t, np.ndarray):
        return _c(t, np.int32)
    return _c(t.detach().cpu().numpy(), np.int32)


class CacheView:
    """Host copy of one paged cache, kept alive while the oracle reads it."""

    def __init__(self, k, v, block_table, num_pages, page_size, num_layers,
                 num_q_heads, num_kv_heads, head_dim):
        self.k = _bf16_bits(k)
        self.v = _bf16_bits(v) if v is not None else None
        self.block_table = _i32(block_table)
        self.struct = _Cache(_ptr(self.k), _ptr(self.v) if self.v is not None else None,
                             _ptr(self.block_table), int(num_pages),
                             int(self.block_table.shape[-1]), int(page_size),
                             int(num_layers), int(num_q_heads), int(num_kv_heads),
                             int(head_dim))


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def slm_row(slm_q, slm: CacheView, batch: int, j: int, b: int, n: int):
    """(s, a, m, lse) of flat SLM head j, sequence b (fp64)."""
    lib = _load()
    q = _bf16_bits(slm_q)
    s = np.zeros(n, np.float64)
    a = np.zeros(n, np.float64)
    m = np.zeros(1, np.float64)
    lse = np.zeros(1, np.float64)
    lib.oracle_slm_row(_ptr(q), ctypes.byref(slm.struct), batch, j, b, n,
                       _ptr(s), _ptr(a), _ptr(m), _ptr(lse))
    return s, a, float(m[0]), float(lse[0])


def split(score, K: int, R: int, M: int):
    """Three-way split of one score row: (crit, marg, recent, counts[K',M',R'])."""
    lib = _load()
    sc = _c(score, np.float64)
    n = sc.shape[0]
    crit = np.zeros(max(K, 1), np.int32)
    marg = np.zeros(max(M, 1), np.int32)
    counts = np.zeros(3, np.int32)
    lib.oracle_split(_ptr(sc), n, K, R, M, _ptr(crit), _ptr(marg), _ptr(counts))
    Kc, Mc, Rc = (int(x) for x in counts)
    return crit[:Kc].copy(), marg[:Mc].copy(), np.arange(n - Rc, n, dtype=np.int32), counts


def select(slm_q, slm: CacheView, seq_lens, rows, k_crit, n_recent, k_marg,
           max_crit: int, max_marg: int, max_n: int):
    """Steps 1-3 for rows x batch.  Returns dict of fp64/int32 arrays indexed
    [row_slot][b]..., row_slot = position of the flat SLM head in `rows`."""
    lib = _load()
    q = _bf16_bits(slm_q)
    sl = _i32(seq_lens)
    rows = _i32(rows)
    B = sl.shape[0]
    nr = rows.shape[0]
    kc, nrc, km = _i32(k_crit), _i32(n_recent), _i32(k_marg)
    a = np.zeros((nr, B, max_n), np.float64)
    s = np.zeros((nr, B, max_n), np.float64)
    stats = np.zeros((nr, B, 2), np.float64)
    crit = np.zeros((nr, B, max(max_crit, 1)), np.int32)
    marg = np.zeros((nr, B, max(max_marg, 1)), np.int32)
    counts = np.zeros((nr, B, 3), np.int32)
    lib.oracle_select(_ptr(q), ctypes.byref(slm.struct), _ptr(sl), B, max_n,
                      _ptr(rows), nr, _ptr(kc), _ptr(nrc), _ptr(km),
                      crit.shape[2], marg.shape[2], _ptr(a), _ptr(s), _ptr(stats),
                      _ptr(crit), _ptr(marg), _ptr(counts))
    return {"a": a, "s": s, "stats": stats, "crit": crit, "marg": marg,
            "counts": counts, "rows": rows}


def select_acc(slm_q, slm: CacheView, seq_lens, rows, k_crit, n_recent, k_marg,
               max_crit: int, max_marg: int, max_n: int, acc: np.ndarray):
    """Variant f1: as `select`, ranking by the running column sums acc (fp64
    [rows][B][max_n], updated in place: acc += a')."""
    lib = _load()
    q = _bf16_bits(slm_q)
    sl = _i32(seq_lens)
    rows = _i32(rows)
    B = sl.shape[0]
    nr = rows.shape[0]
    assert acc.dtype == np.float64 and acc.shape == (nr, B, max_n) and acc.flags.c_contiguous
    kc, nrc, km = _i32(k_crit), _i32(n_recent), _i32(k_marg)
    a = np.zeros((nr, B, max_n), np.float64)
    s = np.zeros((nr, B, max_n), np.float64)
    stats = np.zeros((nr, B, 2), np.float64)
    crit = np.zeros((nr, B, max(max_crit, 1)), np.int32)
    marg = np.zeros((nr, B, max(max_marg, 1)), np.int32)
    counts = np.zeros((nr, B, 3), np.int32)
    lib.oracle_select_acc(_ptr(q), ctypes.byref(slm.struct), _ptr(sl), B, max_n,
                          _ptr(rows), nr, _ptr(kc), _ptr(nrc), _ptr(km),
                          crit.shape[2], marg.shape[2], _ptr(acc), _ptr(a), _ptr(s),
                          _ptr(stats), _ptr(crit), _ptr(marg), _ptr(counts))
    return {"a": a, "s": s, "stats": stats, "crit": crit, "marg": marg,
            "counts": counts, "rows": rows, "acc": acc.copy()}


def attend(layer: int, cache_layer: int, q, llm: CacheView, seq_lens, head_map,
           sel: dict, n_slm_heads: int):
    """Step 4 for one LLM layer given selection dict `sel` (from `select`, or
    the GPU's lists re-packed the same way).  Returns (out[B,H,d], wsum[B,H])."""
    lib = _load()
    qq = _bf16_bits(q)
    sl = _i32(seq_lens)
    hm = _i32(head_map)
    B = sl.shape[0]
    H, d = llm.struct.num_q_heads, llm.struct.head_dim
    row_slot = np.full(n_slm_heads, -1, np.int32)
    for slot, j in enumerate(sel["rows"]):
        row_slot[j] = slot
    a = _c(sel["a"], np.float64)
    crit = _c(sel["crit"], np.int32)
    marg = _c(sel["marg"], np.int32)
    counts = _c(sel["counts"], np.int32)
    out = np.zeros((B, H, d), np.float64)
    wsum = np.zeros((B, H), np.float64)
    lib.oracle_attend(layer, cache_layer, _ptr(qq), ctypes.byref(llm.struct), _ptr(sl), B,
                      _ptr(hm), _ptr(row_slot), _ptr(a), a.shape[2], _ptr(crit),
                      _ptr(marg), _ptr(counts), crit.shape[2], marg.shape[2],
                      _ptr(out), _ptr(wsum))
    return out, wsum


def select_group(layer: int, H: int, H_kv: int, head_map, sel: dict, seq_lens, k_crit,
                 n_recent, k_marg, max_crit: int, max_marg: int, n_slm_heads: int):
    """Variant f2: per-kv-group shared split of F_g = Σ_{h in group} a'_{f(layer,h)}
    (sel from `select` over the image of the head map).  Returns a dict indexed
    [g][b]... with "score", "crit", "marg", "counts"."""
    lib = _load()
    hm = _i32(head_map)
    sl = _i32(seq_lens)
    B = sl.shape[0]
    row_slot = np.full(n_slm_heads, -1, np.int32)
    for slot, j in enumerate(sel["rows"]):
        row_slot[j] = slot
    a = _c(sel["a"], np.float64)
    max_n = a.shape[2]
    kc, nrc, km = _i32(k_crit), _i32(n_recent), _i32(k_marg)
    score = np.zeros((H_kv, B, max_n), np.float64)
    crit = np.zeros((H_kv, B, max(max_crit, 1)), np.int32)
    marg = np.zeros((H_kv, B, max(max_marg, 1)), np.int32)
    counts = np.zeros((H_kv, B, 3), np.int32)
    lib.oracle_select_group(layer, H, H_kv, _ptr(hm), _ptr(row_slot), _ptr(a), max_n, _ptr(sl),
                            B, _ptr(kc), _ptr(nrc), _ptr(km), crit.shape[2], marg.shape[2],
                            _ptr(score), _ptr(crit), _ptr(marg), _ptr(counts))
    return {"score": score, "crit": crit, "marg": marg, "counts": counts}


def attend_group(layer: int, cache_layer: int, q, llm: CacheView, seq_lens, head_map,
                 sel: dict, gsel: dict, n_slm_heads: int):
    """Variant f2 step 4: head h uses its group's shared sets (gsel) and its own
    SLM row's weights (sel["a"]).  Returns (out[B,H,d], wsum[B,H])."""
    lib = _load()
    qq = _bf16_bits(q)
    sl = _i32(seq_lens)
    hm = _i32(head_map)
    B = sl.shape[0]
    H, d = llm.struct.num_q_heads, llm.struct.head_dim
    row_slot = np.full(n_slm_heads, -1, np.int32)
    for slot, j in enumerate(sel["rows"]):
        row_slot[j] = slot
    a = _c(sel["a"], np.float64)
    crit = _c(gsel["crit"], np.int32)
    marg = _c(gsel["marg"], np.int32)
    counts = _c(gsel["counts"], np.int32)
    out = np.zeros((B, H, d), np.float64)
    wsum = np.zeros((B, H), np.float64)
    lib.oracle_attend_group(layer, cache_layer, _ptr(qq), ctypes.byref(llm.struct), _ptr(sl), B,
                            _ptr(hm), _ptr(row_slot), _ptr(a), a.shape[2], _ptr(crit),
                            _ptr(marg), _ptr(counts), crit.shape[2], marg.shape[2],
                            _ptr(out), _ptr(wsum))
    return out, wsum


def match_window(n: int, w_min: int = 100, w_max: int = 200, keep_last: bool = True):
    """Variant f3 window decision (R17): None (DEFER) or (start, len)."""
    lib = _load()
    st, ln = ctypes.c_int32(), ctypes.c_int32()
    ok = lib.oracle_match_window(int(n), int(w_min), int(w_max), int(bool(keep_last)),
                                 ctypes.byref(st), ctypes.byref(ln))
    return (st.value, ln.value) if ok else None


def prefill_scores(q, cache: CacheView, b: int, start: int, length: int) -> np.ndarray:
    """Variant f3: F [L*H][length] (fp64) — Eq. 1 column sums over the window
    [start, start+length) of the causal prefill attention rows of its queries
    q [L][length][H][d] (bf16) against the paged K of sequence b."""
    lib = _load()
    qq = _bf16_bits(q)
    L, H = cache.struct.num_layers, cache.struct.num_q_heads
    F = np.zeros((L * H, length), np.float64)
    lib.oracle_prefill_scores(_ptr(qq), ctypes.byref(cache.struct), int(b), int(start),
                              int(length), _ptr(F))
    return F


def topk_mask(F, k: int) -> np.ndarray:
    lib = _load()
    f = _c(F, np.float64)
    m = np.zeros(f.shape[0], np.uint8)
    lib.oracle_topk(_ptr(f), f.shape[0], k, _ptr(m))
    return m.astype(bool)


def match_heads(llm_F, slm_F, k: int):
    """Eq. 2-3: (head_map[n_llm], jaccard[n_llm])."""
    lib = _load()
    lf = _c(llm_F, np.float64)
    sf = _c(slm_F, np.float64)
    n_llm, w = lf.shape
    n_slm = sf.shape[0]
    hm = np.zeros(n_llm, np.int32)
    jac = np.zeros(n_llm, np.float64)
    lib.oracle_match_heads(_ptr(lf), n_llm, _ptr(sf), n_slm, w, k, _ptr(hm), _ptr(jac))
    return hm, jac


def accumulate_scores(A) -> np.ndarray:
    """Eq. 1 column sums of an n x n attention matrix."""
    lib = _load()
    a = _c(A, np.float64)
    n = a.shape[0]
    F = np.zeros(n, np.float64)
    lib.oracle_accumulate_scores(_ptr(a), n, _ptr(F))
    return F


def image_rows(head_map) -> np.ndarray:
    """Sorted distinct flat SLM heads referenced by the head map."""
    return np.unique(_i32(head_map)).astype(np.int32)
