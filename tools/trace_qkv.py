"""Dev tool: producer CTA timeline (knob "trace") for L chained projections (graph, PDL).
Prints per-layer medians (us) relative to the layer's first CTA start: pdl-wait return, first
stage landed, MMA loop end, first accumulator ready, partials counted, reducer done, exit."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2602_07223_b200 import QkvProjection  # noqa: E402

L, D, Hq, Hkv = int(os.environ.get("LAYERS", 8)), 4096, 32, 8
B, rows = int(os.environ.get("B", 1)), int(os.environ.get("ROWS", 5))
n_out = (Hq + 2 * Hkv) * 128
w = (torch.randn(L, n_out, D, device="cuda") / 64).to(torch.bfloat16)
proj = QkvProjection(w, torch.ones(L, D, device="cuda"), Hq, Hkv)
proj.set_dev_knob("trace", 1)
x = torch.randn(B, rows, D, device="cuda")
pos = torch.full((B,), 32768, dtype=torch.int32, device="cuda")
q = torch.empty(B, Hq, rows, 128, dtype=torch.bfloat16, device="cuda")
k = torch.empty(B, rows, Hkv, 128, dtype=torch.bfloat16, device="cuda")
v = torch.empty_like(k)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    g = torch.cuda.CUDAGraph()
    for l in range(L):
        proj.project(l, x, pos, q, k, v, stream=s)
    reps = int(os.environ.get("REPS", 1))  # REPS > 1 with LAYERS=1: the same (L2-hot) weights again
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            for l in range(L):
                proj.project(l, x, pos, q, k, v, stream=s)
    for _ in range(5):
        g.replay()
torch.cuda.synchronize()
proj.close()
t = np.fromfile("/tmp/sa_qkv_trace.bin", dtype=np.uint64).reshape(L, -1, 32).astype(np.int64)
names = ["start", "pdl", "first", "mma_end", "acc0", "counted", "reduced", "exit", "pre_last", "post_first", "mid", "pdl2", "allpre"]
prev_exit = None
for l in range(L):
    a = t[l]
    t0 = a[:, 0].min()
    cols = []
    for i, n in enumerate(names):
        v_ = a[:, i][a[:, i] > 0] - t0
        cols.append(f"{n}={np.median(v_) / 1e3:6.2f}/{v_.max() / 1e3:6.2f}" if len(v_) else f"{n}=-")
    gap = f" gap_from_prev_exit={(t0 - prev_exit) / 1e3:6.2f}" if prev_exit is not None else ""
    prev_exit = a[:, 7].max()
    print(f"L{l}: span={(a[:, 7].max() - t0) / 1e3:6.2f}us " + " ".join(cols) + gap)
    land = [np.median(a[:, 16 + i][a[:, 16 + i] > 0] - t0) / 1e3 for i in range(16) if (a[:, 16 + i] > 0).any()]
    print("     MMA iteration (median us): " + " ".join(f"{x:.2f}" for x in land))
