"""(needs a dev build: make -C paper_2602_07223_b200/csrc EXTRA_NVFLAGS=-DSA_PIPE_TRACE) Dev tool: per-layer verify CTA timeline inside the config-2 iteration graph (knob "trace").
  SA_ITER_SKIP=6 python tools/trace_iter.py      # verify-only graph
Prints, per layer: first CTA start, median / max main-loop end, median / max CTA end (us, relative
to layer 0's first start)."""
import ctypes
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2602_07223_b200 import COLLECT2, Cache, Runner  # noqa: E402
from paper_2602_07223_b200._lib import lib  # noqa: E402

L = int(os.environ.get("LAYERS", 32))
Hq, Hkv, p0, gamma, D = 32, 8, int(os.environ.get("CTX", 32768)), 4, 128
R = gamma + 1
cache = Cache(L, Hkv, D, p0 + R + 64, page_size=256)
for s in range(0, p0, 2048):
    kk = torch.randn((2048, L * Hkv, D), device="cuda").to(torch.bfloat16)
    cache.append(kk, kk)
r = Runner(cache, Hq, max_rows=R, max_prefix=p0)
r.set_dev_knob("trace", 1)  # dev-only knobs (the library never reads the environment)
if os.environ.get("SA_ITER_SKIP"):
    r.set_dev_knob("iter_skip", int(os.environ["SA_ITER_SKIP"]))
r.set_batch([0], [p0])


def rnd(*s):
    return torch.randn(s, device="cuda").to(torch.bfloat16)


qv, kvn, vvn = rnd(L, 1, Hq, R, D), rnd(L, 1, R, Hkv, D), rnd(L, 1, R, Hkv, D)
qd, kdn, vdn = rnd(gamma, L, 1, Hq, D), rnd(gamma, L, 1, Hkv, D), rnd(gamma, L, 1, Hkv, D)
out_v = torch.empty((L, 1, Hq, R, D), device="cuda")
out_d = torch.empty((gamma, L, 1, Hq, D), device="cuda")
st = torch.cuda.Stream()
args = r.iteration_args(gamma, qv, kvn, vvn, qd, kdn, vdn, out_v, out_d, strategy=COLLECT2, mode=0,
                        scale=1 / math.sqrt(D), use_graph=True)
with torch.cuda.stream(st):
    for _ in range(4):
        r.iteration(args, stream=st)
torch.cuda.synchronize()
path = "/tmp/sa_trace_iter.bin"

assert r.trace_dump(path) == 0
raw = np.fromfile(path, dtype=np.uint64).astype(np.int64)
t0 = None
print(f"{'layer':>5s} {'start':>8s} {'st_med':>8s} {'loop_med':>8s} {'loop_max':>8s} {'end_med':>8s} {'end_max':>8s} {'dt':>7s}"
      "   (arrival->merge_done max, loop_max->end_max)")
prev = None
for l in range(min(L, 64)):
    blk = raw[1024 + l * 16384: 1024 + (l + 1) * 16384].reshape(1024, 16)
    blk = blk[blk[:, 0] > 0]
    if not len(blk):
        continue
    if t0 is None:
        t0 = blk[:, 0].min()
    s0, ml, en = (blk[:, 0] - t0) / 1e3, (blk[:, 2] - t0) / 1e3, (blk[:, 1] - t0) / 1e3
    dt = s0.min() - prev if prev is not None else 0.0
    prev = s0.min()
    arr, mdone = (blk[:, 6] - t0) / 1e3, (blk[:, 9] - t0) / 1e3
    has_m = blk[:, 9] > 0
    extra = f"   {(mdone[has_m].max() - arr[blk[:, 6] > 0].max()) if has_m.any() else float('nan'):6.2f} {en.max() - ml.max():6.2f}"
    print(extra, end="")
    print(f"\r{l:5d} {s0.min():8.2f} {np.median(s0):8.2f} {np.median(ml):8.2f} {ml.max():8.2f} {np.median(en):8.2f} {en.max():8.2f} {dt:7.2f}")
