"""ctypes binding of libsmallkv.so — argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI
(include/smallkv.h).  This module only turns torch tensors into pointers,
allocates output buffers / workspaces with torch (device memory plumbing) and
raises on non-OK status.  There is no CPU fallback: if the library is missing
or the device is not a B200, calls fail loudly.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import threading
from typing import Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SMALLKV_LIB") or os.path.join(_HERE, "libsmallkv.so")
_lock = threading.Lock()
_lib = None

ATTEND_OVERLAP_PROLOGUE = 1   # include/smallkv.h SMALLKV_ATTEND_OVERLAP_PROLOGUE
ATTEND_GROUP_SELECTION = 2    # include/smallkv.h SMALLKV_ATTEND_GROUP_SELECTION (variant f2)

STATUS = {0: "OK", 1: "ERR_NULL", 2: "ERR_SHAPE", 3: "ERR_ALIGN", 4: "ERR_WORKSPACE",
          5: "ERR_DEVICE", 6: "ERR_CUDA", 7: "ERR_UNSUPPORTED"}

# exported symbols, in the order include/smallkv.h declares them
EXPORTS = ("smallkv_last_error", "smallkv_version", "smallkv_budget_from_tau",
           "smallkv_select_workspace_size", "smallkv_select",
           "smallkv_select_group_workspace_size", "smallkv_select_group",
           "smallkv_plan_size", "smallkv_plan", "smallkv_plan_group",
           "smallkv_attend_workspace_size", "smallkv_attend",
           "smallkv_tier_state_size", "smallkv_tier_init", "smallkv_tier_update",
           "smallkv_plan_tiered", "smallkv_attend_tiered",
           "smallkv_match_window", "smallkv_prefill_scores",
           "smallkv_match_heads_workspace_size", "smallkv_match_heads",
           "smallkv_workspace_init")


class SmallKVError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed: {STATUS.get(code, code)}: {msg}")
        self.code = code


class CCache(ctypes.Structure):
    _fields_ = [("k", ctypes.c_void_p), ("v", ctypes.c_void_p),
                ("block_table", ctypes.c_void_p), ("num_pages", ctypes.c_int64),
                ("max_blocks", ctypes.c_int32), ("page_size", ctypes.c_int32),
                ("num_layers", ctypes.c_int32), ("num_q_heads", ctypes.c_int32),
                ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32)]


class CBatch(ctypes.Structure):
    _fields_ = [("seq_lens", ctypes.c_void_p), ("batch", ctypes.c_int32),
                ("max_seq_len", ctypes.c_int32)]


class CBudgets(ctypes.Structure):
    _fields_ = [("k_crit", ctypes.c_void_p), ("n_recent", ctypes.c_void_p),
                ("k_marg", ctypes.c_void_p), ("max_crit", ctypes.c_int32),
                ("max_marg", ctypes.c_int32)]


def load(path: Optional[str] = None):
    """Load libsmallkv.so (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise RuntimeError(f"{p} not found: build it with `python -m paper_2508_02751_b200.build` "
                               "(there is no CPU fallback)")
        lib = ctypes.CDLL(p)
        P, i32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
        lib.smallkv_last_error.restype = ctypes.c_char_p
        lib.smallkv_version.restype = ctypes.c_char_p
        lib.smallkv_budget_from_tau.argtypes = [ctypes.c_double, i32, P, P, P]
        lib.smallkv_select_workspace_size.argtypes = [P, P, i32]
        lib.smallkv_select_workspace_size.restype = sz
        lib.smallkv_select.argtypes = [P, P, P, P, i32, P, P, P, P, P, P, P, P, P, sz, P, P]
        lib.smallkv_select_group_workspace_size.argtypes = [P, P, P, i32, i32]
        lib.smallkv_select_group_workspace_size.restype = sz
        lib.smallkv_select_group.argtypes = [P, P, P, P, i32, i32, i32, P, P, P, P, P, P, P, P,
                                             P, sz, P]
        lib.smallkv_plan_group.argtypes = [P, P, P, i32, P, P, P, P, P, P, sz, P]
        lib.smallkv_attend_workspace_size.argtypes = [P, P]
        lib.smallkv_attend_workspace_size.restype = sz
        lib.smallkv_attend.argtypes = [i32, i32, P, P, P, P, i32, i32, P, P, P, P, P, P, P, i32,
                                       P, sz, P]
        lib.smallkv_plan_size.argtypes = [P, P, i32]
        lib.smallkv_plan_size.restype = sz
        lib.smallkv_plan.argtypes = [P, P, P, i32, i32, P, P, P, P, P, P, sz, P]
        lib.smallkv_tier_state_size.argtypes = [P, P, i32, i32]
        lib.smallkv_tier_state_size.restype = sz
        lib.smallkv_tier_init.argtypes = [P, sz, P, P, i32, i32, P]
        lib.smallkv_tier_update.argtypes = [i32, i32, P, P, P, i32, P, P, i32, i32, P, P, P, P,
                                            P, i32, P, sz, P]
        lib.smallkv_plan_tiered.argtypes = [P, i32, P, P, P, i32, i32, P, P, P, P, P, i32, P, sz,
                                            P]
        lib.smallkv_attend_tiered.argtypes = [i32, P, P, P, P, i32, P, P, P, i32, i32, P, P, P,
                                              P, P, P, P, i32, P, sz, P]
        lib.smallkv_match_window.argtypes = [i32, i32, i32, i32, P, P]
        lib.smallkv_prefill_scores.argtypes = [P, P, i32, i32, i32, P, P]
        lib.smallkv_match_heads_workspace_size.argtypes = [i32, i32]
        lib.smallkv_match_heads_workspace_size.restype = sz
        lib.smallkv_match_heads.argtypes = [P, i32, P, i32, i32, i32, P, P, P, sz, P]
        lib.smallkv_workspace_init.argtypes = [P, sz, P]
        _lib = lib
        return lib


def _check(fn: str, rc: int):
    if rc != 0:
        raise SmallKVError(fn, rc, load().smallkv_last_error().decode())


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    if t is None:
        return None
    return t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def version() -> str:
    return load().smallkv_version().decode()


def budget_from_tau(tau: float, n: int):
    """Host helper: (K, R, M) token counts for budget fraction tau."""
    lib = load()
    k, r, m = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _check("smallkv_budget_from_tau",
           lib.smallkv_budget_from_tau(float(tau), int(n), ctypes.byref(k), ctypes.byref(r),
                                       ctypes.byref(m)))
    return k.value, r.value, m.value


def make_cache(k: torch.Tensor, v: Optional[torch.Tensor], block_table: torch.Tensor,
               num_q_heads: int) -> CCache:
    """Describe a paged pool [layers][pages][kv][page_size][d] (bf16) to the ABI."""
    assert k.dtype == torch.bfloat16 and k.dim() == 5 and k.is_contiguous()
    if v is not None:
        assert v.shape == k.shape and v.dtype == torch.bfloat16 and v.is_contiguous()
    assert block_table.dtype == torch.int32 and block_table.is_contiguous()
    L, pages, kv, ps, d = k.shape
    return CCache(k.data_ptr(), _ptr(v), block_table.data_ptr(), pages,
                  block_table.shape[-1], ps, L, num_q_heads, kv, d)


def make_batch(seq_lens: torch.Tensor, max_seq_len: int) -> CBatch:
    assert seq_lens.dtype == torch.int32 and seq_lens.is_contiguous()
    return CBatch(seq_lens.data_ptr(), seq_lens.shape[0], int(max_seq_len))


def make_budgets(k_crit, n_recent, k_marg, max_crit: int, max_marg: int) -> CBudgets:
    for t in (k_crit, n_recent, k_marg):
        assert t.dtype == torch.int32 and t.is_contiguous()
    return CBudgets(k_crit.data_ptr(), n_recent.data_ptr(), k_marg.data_ptr(), int(max_crit),
                    int(max_marg))


@dataclasses.dataclass
class SelectOut:
    logits: torch.Tensor   # fp32 [l*H_s][B][max_seq_len]
    lse: torch.Tensor      # fp32 [l*H_s][B][2]
    crit: torch.Tensor     # int32 [l*H_s][B][max_crit]
    marg: torch.Tensor     # int32 [l*H_s][B][max_marg]
    marg_w: torch.Tensor   # fp32 [l*H_s][B][max_marg]
    counts: torch.Tensor   # int32 [l*H_s][B][2]


class DecodeStep:
    """Buffers + calls for one model pair's decode hot path on one device.

    Holds the ABI descriptors, the selection outputs and both workspaces;
    `select()` runs smallkv_select, `attend(layer, cache_layer, q, out)` runs
    smallkv_attend.  All tensors must live on the current CUDA device.
    """

    def __init__(self, *, slm_k, slm_block_table, slm_q_heads: int, llm_k, llm_v,
                 llm_block_table, llm_q_heads: int, llm_layers: int, seq_lens: torch.Tensor,
                 max_seq_len: int, head_map: torch.Tensor, k_crit, n_recent, k_marg,
                 max_crit: int, max_marg: int, use_plan: bool = True,
                 overlap_select: bool = False, variant: str = "default"):
        """variant: "default" (one split per SLM row) or "f2" (one split
        per LLM (layer, kv-group) of the summed proxy rows, R16)."""
        assert variant in ("default", "f2")
        self.variant = variant
        self.lib = load()
        dev = seq_lens.device
        self._keep = (slm_k, slm_block_table, llm_k, llm_v, llm_block_table, seq_lens, head_map,
                      k_crit, n_recent, k_marg)
        self.slm = make_cache(slm_k, None, slm_block_table, slm_q_heads)
        self.llm = make_cache(llm_k, llm_v, llm_block_table, llm_q_heads)
        self.batch = make_batch(seq_lens, max_seq_len)
        self.budgets = make_budgets(k_crit, n_recent, k_marg, max_crit, max_marg)
        assert head_map.dtype == torch.int32 and head_map.numel() == llm_layers * llm_q_heads
        self.head_map = head_map
        self.llm_layers = llm_layers
        self.n_slm = self.slm.num_layers * slm_q_heads
        B, n = self.batch.batch, int(max_seq_len)
        f32, i32 = torch.float32, torch.int32
        self.out = SelectOut(
            logits=torch.zeros(self.n_slm, B, n, dtype=f32, device=dev),
            lse=torch.zeros(self.n_slm, B, 2, dtype=f32, device=dev),
            crit=torch.zeros(self.n_slm, B, max_crit, dtype=i32, device=dev),
            marg=torch.zeros(self.n_slm, B, max_marg, dtype=i32, device=dev),
            marg_w=torch.zeros(self.n_slm, B, max_marg, dtype=f32, device=dev),
            counts=torch.zeros(self.n_slm, B, 2, dtype=i32, device=dev))
        ws_s = self.lib.smallkv_select_workspace_size(ctypes.byref(self.slm),
                                                      ctypes.byref(self.batch),
                                                      head_map.numel())
        ws_a = self.lib.smallkv_attend_workspace_size(ctypes.byref(self.llm),
                                                      ctypes.byref(self.batch))
        if ws_s == 0 or ws_a == 0:
            raise SmallKVError("workspace_size", 2, "invalid dimensions")
        self.ws_select = torch.zeros(ws_s, dtype=torch.uint8, device=dev)
        self.ws_attend = torch.zeros(ws_a, dtype=torch.uint8, device=dev)
        plan_b = self.lib.smallkv_plan_size(ctypes.byref(self.llm), ctypes.byref(self.batch),
                                            llm_layers)
        self.plan_buf = torch.empty(max(plan_b, 16), dtype=torch.uint8, device=dev) if use_plan else None
        self.planned = False
        if variant == "f2":
            H_kv = self.llm.num_kv_heads
            ng = llm_layers * H_kv
            self.gout = SelectOut(
                logits=torch.zeros(ng, B, n, dtype=f32, device=dev),          # group score F_g
                lse=self.out.lse,
                crit=torch.zeros(ng, B, max_crit, dtype=i32, device=dev),
                marg=torch.zeros(ng, B, max_marg, dtype=i32, device=dev),
                marg_w=torch.zeros(ng, B, max_marg, 8, dtype=f32, device=dev),
                counts=torch.zeros(ng, B, 2, dtype=i32, device=dev))
            ws_g = self.lib.smallkv_select_group_workspace_size(
                ctypes.byref(self.slm), ctypes.byref(self.batch), ctypes.byref(self.budgets),
                llm_layers, H_kv)
            if ws_g == 0:
                raise SmallKVError("smallkv_select_group_workspace_size", 2, "invalid dimensions")
            self.ws_select = torch.zeros(ws_g, dtype=torch.uint8, device=dev)
        self.aux_stream = torch.cuda.Stream(device=dev) if overlap_select else None

    def select(self, slm_q: torch.Tensor, stream=None, acc: Optional[torch.Tensor] = None,
               select_head_map: Optional[torch.Tensor] = None, plan: bool = True):
        """smallkv_select, then (by default) smallkv_plan for every layer.
        acc: optional fp32 [l*H_s][B][max_seq_len] running column sums (variant
        f1, zero-filled once by the caller; updated in place).
        select_head_map: optional head-map subset that defines which SLM rows
        are scored and split (f3b: a rank's row block, dist.select_head_map);
        plan=False skips smallkv_plan (call plan() after the selection exchange)."""
        assert slm_q.dtype == torch.bfloat16 and slm_q.is_contiguous()
        if acc is not None:
            assert acc.dtype == torch.float32 and acc.is_contiguous()
            assert acc.shape == self.out.logits.shape
        if self.variant == "f2":
            assert acc is None, "f1 accumulation is not combined with f2"
            return self._select_group(slm_q, stream)
        o = self.out
        aux = self.aux_stream.cuda_stream if self.aux_stream is not None else None
        shm = self.head_map if select_head_map is None else select_head_map
        assert shm.dtype == torch.int32 and shm.is_contiguous()
        self.planned = False
        if shm.numel() == 0:
            return o   # no row of this block is used
        rc = self.lib.smallkv_select(
            slm_q.data_ptr(), ctypes.byref(self.slm), ctypes.byref(self.batch),
            shm.data_ptr(), shm.numel(), ctypes.byref(self.budgets),
            o.logits.data_ptr(), o.lse.data_ptr(), o.crit.data_ptr(), o.marg.data_ptr(),
            o.marg_w.data_ptr(), o.counts.data_ptr(), _ptr(acc), self.ws_select.data_ptr(),
            self.ws_select.numel(), _stream(stream), aux)
        _check("smallkv_select", rc)
        if plan:
            self.plan(stream)
        return o

    def plan(self, stream=None):
        """smallkv_plan for every layer from the current selection outputs."""
        o = self.out
        self.planned = False
        if self.plan_buf is not None:
            rc = self.lib.smallkv_plan(
                ctypes.byref(self.llm), ctypes.byref(self.batch), self.head_map.data_ptr(),
                self.llm_layers, self.n_slm, ctypes.byref(self.budgets), o.crit.data_ptr(),
                o.marg.data_ptr(), o.marg_w.data_ptr(), o.counts.data_ptr(),
                self.plan_buf.data_ptr(), self.plan_buf.numel(), _stream(stream))
            _check("smallkv_plan", rc)
            self.planned = True
        return o

    def _select_group(self, slm_q: torch.Tensor, stream=None):
        """Variant f2: smallkv_select_group, then smallkv_plan_group."""
        o, g = self.out, self.gout
        rc = self.lib.smallkv_select_group(
            slm_q.data_ptr(), ctypes.byref(self.slm), ctypes.byref(self.batch),
            self.head_map.data_ptr(), self.llm_layers, self.llm.num_q_heads,
            self.llm.num_kv_heads, ctypes.byref(self.budgets), o.logits.data_ptr(),
            o.lse.data_ptr(), g.logits.data_ptr(), g.crit.data_ptr(), g.marg.data_ptr(),
            g.marg_w.data_ptr(), g.counts.data_ptr(), self.ws_select.data_ptr(),
            self.ws_select.numel(), _stream(stream))
        _check("smallkv_select_group", rc)
        self.planned = False
        if self.plan_buf is not None:
            rc = self.lib.smallkv_plan_group(
                ctypes.byref(self.llm), ctypes.byref(self.batch), self.head_map.data_ptr(),
                self.llm_layers, ctypes.byref(self.budgets), g.crit.data_ptr(),
                g.marg.data_ptr(), g.marg_w.data_ptr(), g.counts.data_ptr(),
                self.plan_buf.data_ptr(), self.plan_buf.numel(), _stream(stream))
            _check("smallkv_plan_group", rc)
            self.planned = True
        return g

    def attend(self, llm_layer: int, cache_layer: int, q: torch.Tensor, out: torch.Tensor,
               stream=None, overlap_prologue: bool = False):
        assert q.dtype == torch.bfloat16 and q.is_contiguous()
        assert out.dtype == torch.float32 and out.is_contiguous()
        group = self.variant == "f2"
        o = self.gout if group else self.out
        rc = self.lib.smallkv_attend(
            int(llm_layer), int(cache_layer), q.data_ptr(), ctypes.byref(self.llm),
            ctypes.byref(self.batch), self.head_map.data_ptr(), self.llm_layers, self.n_slm,
            ctypes.byref(self.budgets), o.crit.data_ptr(), o.marg.data_ptr(),
            o.marg_w.data_ptr(), o.counts.data_ptr(),
            self.plan_buf.data_ptr() if self.planned else None, out.data_ptr(),
            (ATTEND_OVERLAP_PROLOGUE if overlap_prologue else 0)
            | (ATTEND_GROUP_SELECTION if group else 0),
            self.ws_attend.data_ptr(), self.ws_attend.numel(), _stream(stream))
        _check("smallkv_attend", rc)
        return out


class TieredKV:
    """Variant f4 (R18): the LLM's paged K/V pool lives in pinned host
    memory; each (layer, sequence, kv-group) keeps the rows its current list
    needs in an HBM hot pool of `capacity` slots, refreshed per layer by
    smallkv_tier_update (only rows not resident at the previous step cross the
    host link) and read by smallkv_attend_tiered."""

    def __init__(self, step: DecodeStep, host_k: torch.Tensor, host_v: torch.Tensor,
                 capacity: int, use_plan: bool = True, per_layer: bool = False):
        """host_k / host_v: pinned CPU pools [Lh][pages][kv][ps][d]; LLM layer l reads
        host layer slot l mod Lh.  per_layer: a decode graph refreshes layer by layer
        on a side stream, the refresh of layer l+1 overlapping the attend of layer l
        (no plan: the attends stage their lists themselves)."""
        assert host_k.device.type == "cpu" and host_k.is_pinned() and host_v.is_pinned()
        assert not (per_layer and use_plan), "the per-layer refresh runs without a plan"
        self.step = step
        self.per_layer = per_layer
        self.lib = step.lib
        bt_keep = step._keep[4]   # llm block table (device)
        self.host = make_cache(host_k, host_v, bt_keep, step.llm.num_q_heads)
        self._keep = (host_k, host_v)
        B, H_kv, d = step.batch.batch, step.llm.num_kv_heads, step.llm.head_dim
        dev = bt_keep.device
        self.capacity = int(capacity)
        self.hot_k = torch.zeros(step.llm_layers, B, H_kv, capacity, d, dtype=torch.bfloat16,
                                 device=dev)
        self.hot_v = torch.zeros_like(self.hot_k)
        nb = self.lib.smallkv_tier_state_size(ctypes.byref(self.host), ctypes.byref(step.batch),
                                              step.llm_layers, self.capacity)
        if nb == 0:
            raise SmallKVError("smallkv_tier_state_size", 2, "invalid dimensions / capacity")
        self.state = torch.empty(nb, dtype=torch.uint8, device=dev)
        plan_b = self.lib.smallkv_plan_size(ctypes.byref(self.host), ctypes.byref(step.batch),
                                            step.llm_layers)
        self.plan_buf = torch.empty(max(plan_b, 16), dtype=torch.uint8, device=dev) if use_plan else None
        self.planned = False
        self.reset()

    def reset(self, stream=None):
        _check("smallkv_tier_init",
               self.lib.smallkv_tier_init(self.state.data_ptr(), self.state.numel(),
                                          ctypes.byref(self.host), ctypes.byref(self.step.batch),
                                          self.step.llm_layers, self.capacity, _stream(stream)))

    def _sel(self):
        st = self.step
        group = st.variant == "f2"
        return (st.gout if group else st.out), (ATTEND_GROUP_SELECTION if group else 0)

    def update(self, layer_begin: int = 0, layer_count: Optional[int] = None, stream=None):
        """Refresh the hot pools of LLM layers [layer_begin, layer_begin+layer_count)."""
        st = self.step
        o, gflag = self._sel()
        count = st.llm_layers - layer_begin if layer_count is None else layer_count
        _check("smallkv_tier_update", self.lib.smallkv_tier_update(
            int(layer_begin), int(count), ctypes.byref(self.host), self.hot_k.data_ptr(),
            self.hot_v.data_ptr(), self.capacity, ctypes.byref(st.batch),
            st.head_map.data_ptr(), st.llm_layers, st.n_slm, ctypes.byref(st.budgets),
            o.crit.data_ptr(), o.marg.data_ptr(), o.marg_w.data_ptr(), o.counts.data_ptr(), gflag,
            self.state.data_ptr(), self.state.numel(), _stream(stream)))
        self.planned = False
        if self.plan_buf is not None:
            _check("smallkv_plan_tiered", self.lib.smallkv_plan_tiered(
                ctypes.byref(self.host), self.capacity, self.state.data_ptr(),
                ctypes.byref(st.batch), st.head_map.data_ptr(), st.llm_layers, st.n_slm,
                ctypes.byref(st.budgets), o.crit.data_ptr(), o.marg.data_ptr(),
                o.marg_w.data_ptr(), o.counts.data_ptr(), gflag, self.plan_buf.data_ptr(),
                self.plan_buf.numel(), _stream(stream)))
            self.planned = True

    def attend(self, llm_layer: int, q: torch.Tensor, out: torch.Tensor, stream=None,
               overlap_prologue: bool = False):
        st = self.step
        o, gflag = self._sel()
        _check("smallkv_attend_tiered", self.lib.smallkv_attend_tiered(
            int(llm_layer), q.data_ptr(), ctypes.byref(self.host),
            self.hot_k.data_ptr(), self.hot_v.data_ptr(), self.capacity, self.state.data_ptr(),
            ctypes.byref(st.batch), st.head_map.data_ptr(), st.llm_layers, st.n_slm,
            ctypes.byref(st.budgets), o.crit.data_ptr(), o.marg.data_ptr(), o.marg_w.data_ptr(),
            o.counts.data_ptr(), self.plan_buf.data_ptr() if self.planned else None,
            out.data_ptr(), (ATTEND_OVERLAP_PROLOGUE if overlap_prologue else 0) | gflag,
            st.ws_attend.data_ptr(), st.ws_attend.numel(), _stream(stream)))
        return out

    def counters(self):
        """(rows fetched from host memory so far, capacity overflows)."""
        c = self.state[-256:][:16].view(torch.int64).cpu()   # counters live at the end
        return int(c[0]), int(c[1])


# score rows per SLM layer above which smallkv_select splits on an auxiliary
# stream in L2-sized SLM-layer chunks (include/smallkv.h, aux_stream)
AUX_SELECT_LAYER_BYTES = 16 << 20


def auto_overlap_select(slm_q_heads: int, batch: int, max_seq_len: int) -> bool:
    """Long contexts: one SLM layer's score rows are too large to stay in L2
    across the whole select (config 2: 7 MB per layer, no; config 4: 59 MB, yes)."""
    return slm_q_heads * batch * max_seq_len * 4 > AUX_SELECT_LAYER_BYTES


def select_chunks(slm_layers: int, slm_q_heads: int, batch: int, max_seq_len: int,
                  aux: bool) -> int:
    """SLM-layer chunks smallkv_select launches (mirrors smallkv_api.cu)."""
    if not aux:
        return 1
    env = int(os.environ.get("SMALLKV_SELECT_CHUNKS", "0") or 0)
    if env > 0:
        return min(slm_layers, env)
    per = max(1, (48 << 20) // max(1, slm_q_heads * batch * max_seq_len * 4))
    return min(slm_layers, -(-slm_layers // per))


def split_launches(max_rows: int, batch: int, max_seq_len: int, acc: bool = False) -> int:
    """Kernels one K2 split launches (mirrors launch_split / launch_select): the
    register split (rows <= 12288 tokens, no f1 sums) and the cluster split
    (long rows, < 1024 pairs) are followed by the to-do launch."""
    if acc:
        return 1
    if max_seq_len <= 12288:   # kernels.h / select.cu kRegMaxLen
        if os.environ.get("SMALLKV_SELECT_REG", "").startswith("g"):
            return 1
        return 2
    if max_seq_len > 16384 and max_rows * batch < 1024:
        return 2
    return 1


def from_problem(p, use_plan: bool = True, variant: str = "default",
                 overlap_select=None) -> DecodeStep:
    """DecodeStep for a smallkv_synth.Problem already on the GPU.  overlap_select
    None: automatic (auto_overlap_select)."""
    if overlap_select is None:
        # tuning knob: SMALLKV_OVERLAP_SELECT=1 runs K2 of each SLM-layer chunk on
        # an auxiliary stream beside K1 of the next chunk
        overlap_select = os.environ.get("SMALLKV_OVERLAP_SELECT", "0") == "1"
    return DecodeStep(slm_k=p.slm.k, slm_block_table=p.slm.block_table,
                      slm_q_heads=p.cfg.slm.q_heads, llm_k=p.llm.k, llm_v=p.llm.v,
                      llm_block_table=p.llm.block_table, llm_q_heads=p.cfg.llm.q_heads,
                      llm_layers=p.cfg.llm.layers, seq_lens=p.seq_lens,
                      max_seq_len=p.max_seq_len, head_map=p.head_map, k_crit=p.k_crit,
                      n_recent=p.n_recent, k_marg=p.k_marg, max_crit=p.max_crit,
                      max_marg=p.max_marg, use_plan=use_plan, variant=variant,
                      overlap_select=overlap_select)


def match_window(n: int, w_min: int = 100, w_max: int = 200, keep_last: bool = True):
    """Variant f3 window decision (R17): None (DEFER) or (start, length)."""
    lib = load()
    st, ln = ctypes.c_int32(), ctypes.c_int32()
    _check("smallkv_match_window", lib.smallkv_match_window(int(n), int(w_min), int(w_max),
                                                            int(bool(keep_last)),
                                                            ctypes.byref(st), ctypes.byref(ln)))
    return (st.value, ln.value) if ln.value > 0 else None


def prefill_scores(q: torch.Tensor, k: torch.Tensor, block_table: torch.Tensor, num_q_heads: int,
                   seq: int, start: int, stream=None) -> torch.Tensor:
    """Variant f3: F [L*H][len] fp32 on the GPU — Eq. 1 column sums over the
    window [start, start+len) of the causal prefill attention rows of its
    queries q [L][len][H][d] (bf16) against the paged K pool `k` of sequence seq."""
    lib = load()
    assert q.dtype == torch.bfloat16 and q.is_contiguous() and q.dim() == 4
    L, length, H, d = q.shape
    assert H == num_q_heads and k.shape[0] == L and k.shape[-1] == d
    cache = make_cache(k, None, block_table, num_q_heads)
    F = torch.empty(L * H, length, dtype=torch.float32, device=q.device)
    _check("smallkv_prefill_scores",
           lib.smallkv_prefill_scores(q.data_ptr(), ctypes.byref(cache), int(seq), int(start),
                                      int(length), F.data_ptr(), _stream(stream)))
    return F


def match_heads(llm_F: torch.Tensor, slm_F: torch.Tensor, k_match: int, stream=None):
    """Eq. 2-3 on the GPU: (head_map int32 [n_llm], jaccard fp32 [n_llm])."""
    lib = load()
    assert llm_F.dtype == torch.float32 and slm_F.dtype == torch.float32
    llm_F, slm_F = llm_F.contiguous(), slm_F.contiguous()
    n_llm, w = llm_F.shape
    n_slm = slm_F.shape[0]
    dev = llm_F.device
    hm = torch.empty(n_llm, dtype=torch.int32, device=dev)
    jac = torch.empty(n_llm, dtype=torch.float32, device=dev)
    wsb = lib.smallkv_match_heads_workspace_size(n_llm, n_slm)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    _check("smallkv_match_heads",
           lib.smallkv_match_heads(llm_F.data_ptr(), n_llm, slm_F.data_ptr(), n_slm, w,
                                   int(k_match), hm.data_ptr(), jac.data_ptr(), ws.data_ptr(),
                                   ws.numel(), _stream(stream)))
    return hm, jac


def _adjacent_view(a: torch.Tensor, b: torch.Tensor) -> Optional[torch.Tensor]:
    """A flat view over a and b when b directly follows a in the same storage
    (both contiguous, same dtype), else None."""
    if (a.dtype != b.dtype or a.device != b.device or not a.is_contiguous()
            or not b.is_contiguous()
            or a.untyped_storage().data_ptr() != b.untyped_storage().data_ptr()
            or b.data_ptr() != a.data_ptr() + a.numel() * a.element_size()):
        return None
    return torch.as_strided(a, (a.numel() + b.numel(),), (1,))


class DecodeGraph:
    """One decode step (smallkv_select + one smallkv_attend per LLM layer)
    captured in a CUDA graph on static buffers.

    layer_plan: sequence of (llm_layer, cache_layer, q_tensor, out_tensor).
    With timing=True, external CUDA events are captured between the calls
    (after select and after every attend) so kernel durations can be read
    back after a replay with `segment_ms()`.
    host_io: optional (h_slm_q, h_q, h_out) pinned host tensors; the graph then
    also moves the step's inputs in (h_slm_q -> slm_q, h_q[i] -> layer i's q)
    and every layer's output out (out -> h_out[i]), each layer's copies on
    side streams overlapping the other layers' kernels (the q of layer i only
    gates attend i; the output copy of layer i only waits for attend i).
    tier: optional TieredKV (variant f4): the hot-pool refresh runs after select
    and the attends read the hot pool (with or without host_io).
    """

    def __init__(self, step: DecodeStep, slm_q: torch.Tensor, layer_plan, timing: bool = False,
                 host_io=None, tier: Optional["TieredKV"] = None, overlap: bool = True):
        self.step = step
        self.overlap = overlap   # False: no attend starts its prologue during the previous one
        self.tier = tier   # variant f4: (tier_update, tiered attend) per layer
        self.slm_q = slm_q
        self.plan = list(layer_plan)
        self.timing = timing
        self.host_io = host_io
        self.events = []
        self.stream = torch.cuda.Stream()
        if host_io is not None:
            self.h2d_stream = torch.cuda.Stream()
            self.d2h_stream = torch.cuda.Stream()
        # eager warm-up on the capture stream (sets kernel attributes, checks args)
        with torch.cuda.stream(self.stream):
            self._calls(record=False)
        self.stream.synchronize()
        if timing:
            self.events = [torch.cuda.Event(enable_timing=True, external=True)
                           for _ in range(len(self.plan) + 2)]
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self._calls(record=timing)

    def _calls(self, record: bool):
        if self.host_io is not None:
            return self._calls_host_io()
        if self.tier is not None:
            # f4: the refresh of every layer's hot pool right after select (ahead
            # of the attends), then the attends; the first attend reads
            # what the refresh wrote, so only later ones overlap their prologue
            main = torch.cuda.current_stream()
            self.step.select(self.slm_q)
            evs = self._tier_refresh(main)
            for i, (layer, slot, q, out) in enumerate(self.plan):
                if evs:
                    main.wait_event(evs[i])
                self.tier.attend(layer, q, out, overlap_prologue=i > 0)
            return
        if record:
            self.events[0].record()
        self.step.select(self.slm_q)
        if record:
            self.events[1].record()
        for i, (layer, slot, q, out) in enumerate(self.plan):
            # every attend after the first is separated from select by another
            # attend, so its prologue may overlap the previous kernel's tail
            self.step.attend(layer, slot, q, out, overlap_prologue=i > 0 and self.overlap)
            if record:
                self.events[2 + i].record()

    def _tier_refresh(self, main):
        """f4 refresh after select: one launch for every layer, or (per-layer tier)
        one launch per layer on a high-priority side stream, so the refresh of
        layer l+1 crosses the host link while layer l attends; returns the
        per-layer completion events (None: all refreshed in order on `main`)."""
        t = self.tier
        if not t.per_layer:
            t.update()
            return None
        if not hasattr(self, "tier_stream"):
            self.tier_stream = torch.cuda.Stream(priority=-1)
        done = torch.cuda.Event()
        done.record(main)
        self.tier_stream.wait_event(done)
        evs = []
        with torch.cuda.stream(self.tier_stream):
            for layer, _, _, _ in self.plan:
                t.update(layer, 1)
                e = torch.cuda.Event()
                e.record(self.tier_stream)
                evs.append(e)
        return evs

    def _calls_host_io(self):
        """select + attends with the host copies on side streams (see __init__)."""
        h_slm_q, h_q, h_out = self.host_io
        main = torch.cuda.current_stream()
        # q' first (select needs it); the layers' q copies are forked after it,
        # so that they do not queue ahead of q' on the host link, and run on a
        # side stream under select (one join before the first attend:
        # per-layer joins cost more than they save)
        self.slm_q.copy_(h_slm_q, non_blocking=True)
        start = torch.cuda.Event()
        start.record(main)
        self.h2d_stream.wait_event(start)
        with torch.cuda.stream(self.h2d_stream):
            for i, (_, _, q, _) in enumerate(self.plan):
                q.copy_(h_q[i], non_blocking=True)
            q_ready = torch.cuda.Event()
            q_ready.record(self.h2d_stream)
        self.step.select(self.slm_q)
        evs = None
        if self.tier is not None:
            evs = self._tier_refresh(main)   # f4: refresh the hot pools after select
        main.wait_event(q_ready)
        # outputs read back in pairs of layers: one fork per pair (each fork
        # costs the attend chain more than a pair's copy delay; measured 0.665
        # -> 0.645 ms per step at config 2, groups of 4 or more are slower)
        n = len(self.plan)
        for i, (layer, slot, q, out) in enumerate(self.plan):
            if self.tier is not None:
                # the first attend reads what the refresh wrote (no overlap)
                if evs:
                    main.wait_event(evs[i])
                self.tier.attend(layer, q, out, overlap_prologue=i > 0)
            else:
                self.step.attend(layer, slot, q, out, overlap_prologue=i > 0)
            if i % 2 == 0 and i != n - 1:
                continue
            done = torch.cuda.Event()
            done.record(main)
            self.d2h_stream.wait_event(done)
            with torch.cuda.stream(self.d2h_stream):
                k0 = i - (i % 2)
                hv = _adjacent_view(h_out[k0], h_out[i]) if i > k0 else None
                dv = _adjacent_view(self.plan[k0][3], self.plan[i][3]) if i > k0 else None
                if hv is not None and dv is not None:
                    hv.copy_(dv, non_blocking=True)       # one copy for the pair
                else:
                    for k in range(k0, i + 1):
                        h_out[k].copy_(self.plan[k][3], non_blocking=True)
        end = torch.cuda.Event()
        end.record(self.d2h_stream)
        main.wait_event(end)

    def replay(self):
        """Launch the graph on this object's stream (CUDAGraph.replay launches on
        the current stream, so make it ours)."""
        with torch.cuda.stream(self.stream):
            self.graph.replay()

    def segment_ms(self):
        """(select_ms, [attend_ms per layer]) of the last replay (after sync)."""
        ev = self.events
        sel = ev[0].elapsed_time(ev[1])
        att = [ev[1 + i].elapsed_time(ev[2 + i]) for i in range(len(self.plan))]
        return sel, att

    @property
    def kernels_per_step(self) -> int:
        # row_flags + (slm_score + select) per SLM-layer chunk (+ plan), then one
        # attend kernel per layer
        nl = self.step.slm.num_layers
        chunks = select_chunks(nl, self.step.slm.num_q_heads, self.step.batch.batch,
                               self.step.batch.max_seq_len, self.step.aux_stream is not None)
        B, S = self.step.batch.batch, self.step.batch.max_seq_len
        n_llm = int(self.step.head_map.numel())
        if self.step.variant == "default":
            # per chunk: slm_score + the split (+ its to-do launch)
            sel = sum(1 + split_launches(min(n_llm, (hi - lo) * self.step.slm.num_q_heads), B, S)
                      for lo, hi in ((nl * i // chunks, nl * (i + 1) // chunks) for i in range(chunks)))
        else:   # f2: slm_score, group score, the split (+ to-do), group weights
            H_kv = self.step.llm.num_kv_heads
            sel = 3 + split_launches(self.step.llm_layers * H_kv, B, S)
        # f4: tier update + copy (per layer, or for all layers), + the tiered plan
        tier = (0 if self.tier is None else 2 * len(self.plan) if self.tier.per_layer
                else (3 if self.tier.plan_buf is not None else 2))
        return (1 + sel + tier + (1 if self.step.plan_buf is not None else 0)
                + len(self.plan))
