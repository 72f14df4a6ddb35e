"""SmallKV (arXiv 2508.02751) decode hot path for B200 (sm_100a).

The product is libsmallkv.so (C ABI in include/smallkv.h, CUDA kernels in
csrc/); `smallkv` is its thin ctypes binding.  Build with
`python -m paper_2508_02751_b200.build`.
"""
from . import smallkv  # noqa: F401
from .smallkv import DecodeStep, budget_from_tau, from_problem, match_heads  # noqa: F401
