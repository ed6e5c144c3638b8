"""(needs a dev build: make -C paper_2602_07223_b200/csrc EXTRA_NVFLAGS=-DSA_PIPE_TRACE) Dev tool: verify tail anatomy inside the config-2 iteration graph (knob "trace", verify-only).
For each layer and unit, times (us) relative to the unit's median main-loop end of: the last main-loop
end, the last arrival's PV done / partial stored / arrival counted, the mergers' merge done, and the
CTA ends; printed as medians over units and layers (layers 2.. of the chain)."""
import ctypes
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SA_ITER_SKIP", "6")  # tool parameter -> knob iter_skip
import torch  # noqa: E402

from paper_2602_07223_b200 import COLLECT2, Cache, Runner  # noqa: E402
from paper_2602_07223_b200._lib import lib  # noqa: E402

L = int(os.environ.get("LAYERS", 32))
Hq, Hkv, p0, gamma, D = 32, 8, 32768, 4, 128
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
path = "/tmp/sa_trace_tail.bin"
assert r.trace_dump(path) == 0
raw = np.fromfile(path, dtype=np.uint64).astype(np.int64)
rows = []
for l in range(2, min(L, 64)):
    blk = raw[1024 + l * 16384: 1024 + (l + 1) * 16384].reshape(1024, 16)
    live = blk[:, 0] > 0
    if not live.any():
        continue
    idx = np.nonzero(live)[0]
    splits = (blk[idx, 3] >> 32).max() + 1
    for u in range(int(idx.max() // splits) + 1):
        cta = idx[(idx // splits) == u]
        if len(cta) < splits:
            continue
        b = blk[cta]
        ref = np.median(b[:, 2])
        last = b[np.argmax(b[:, 6])] if (b[:, 6] > 0).any() else None
        md = b[:, 9][b[:, 9] > 0]
        f7 = b[:, 7][b[:, 7] > 0]
        f8 = b[:, 8][b[:, 8] > 0]
        rows.append([b[:, 2].max() - ref, last[4] - ref, last[10] - ref, last[11] - ref, last[12] - ref,
                     last[5] - ref, last[6] - ref,
                     (f7.max() - ref) if len(f7) else np.nan, (f8.max() - ref) if len(f8) else np.nan,
                     (md.max() - ref) if len(md) else np.nan, b[:, 1].max() - ref, b[:, 0].max() - ref])
a = np.array(rows) / 1e3
names = ["loop_end_max", "last:pv_done", "last:l_reduced", "last:ml_stored", "last:o_stored",
         "last:partial_stored", "last:published", "merger:all_flags_seen", "merger:partials_landed",
         "merge_done_max", "cta_end_max", "cta_start_max"]
for i, n in enumerate(names):
    print(f"{n:22s} median {np.nanmedian(a[:, i]):7.2f}  p90 {np.nanpercentile(a[:, i], 90):7.2f} us")
