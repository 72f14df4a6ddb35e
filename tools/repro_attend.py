"""Attend parity on a long list with many staging batches per CTA (diagnostics).

    SMALLKV_ATTEND_CTAS=1 python tools/repro_attend.py [n] [B]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import smallkv_synth as synth  # noqa: E402
from tests import parity  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
B = int(sys.argv[2]) if len(sys.argv) > 2 else 2
H = int(sys.argv[3]) if len(sys.argv) > 3 else 16
cfg = synth.small_config(llm=(1, H, 8, 128), slm=(1, 14, 2, 64), seq_len=n, batch=B,
                         budget=(n // 10, n // 20, n // 10))
p = synth.make_problem(cfg, seed=5, page_size=64).to("cuda")
step, sel_gpu, outs = parity.run_gpu_step(p)
pc = p.to("cpu")
sel = parity.oracle_select(pc)
sg = parity.sel_from_gpu(pc, sel_gpu, sel)
e, ref = parity.compare_attend(pc, 0, outs[0].cpu(), sg)
o = outs[0].cpu().double().numpy()
err = parity.row_normwise(o, ref)
print("n", n, "B", B, "ctas", parity.attend_split(step), "max row-normwise err", float(err.max()),
      "rows > 1e-4:", int((err > 1e-4).sum()), "of", err.size, flush=True)
bad = np.argwhere(err > 1e-4)
print("bad (b, h):", bad[:20].tolist())
