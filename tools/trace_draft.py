"""Dev tool: per-CTA phase timestamps of one draft launch (config-2 shapes)."""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SA_TRACE"] = "1"
import torch  # noqa: E402

from paper_2602_07223_b200 import Cache, Runner  # noqa: E402

L, Hq, Hkv, p0, R, D = 2, 32, 8, 32768, 5, 128
cache = Cache(L, Hkv, D, p0 + 64)
for s in range(0, p0, 4096):
    kk = torch.randn((4096, L * Hkv, D), device="cuda").to(torch.bfloat16)
    cache.append(kk, kk)
r = Runner(cache, Hq, max_rows=R, max_prefix=p0)
r.set_batch([0], [p0])
q = torch.randn((1, Hq, R, D), device="cuda").to(torch.bfloat16)
kn = torch.randn((1, R, Hkv, D), device="cuda").to(torch.bfloat16)
out = torch.empty((1, Hq, R, D), device="cuda")
for l in range(L):
    r.verify(l, q, out, kn, kn, 1 / math.sqrt(D))
    r.select(l)
qd = torch.randn((1, Hq, D), device="cuda").to(torch.bfloat16)
od = torch.empty((1, Hq, D), device="cuda")
for it in range(4):
    if it == 3:
        os.environ["SA_DTRACE_DUMP"] = os.path.join(ROOT, "gpurun_out", "dtrace.bin")
    r.draft(it % L, 2, qd, od, kn[:, 0].contiguous(), kn[:, 0].contiguous())
torch.cuda.synchronize()
tr = np.fromfile(os.path.join(ROOT, "gpurun_out", "dtrace.bin"), dtype=np.uint64).astype(np.int64).reshape(512, 8)
tr = tr[tr[:, 0] > 0]
g0 = tr[:, 0].min()
ph = ["start", "loaded", "computed", "partial", "end"]
print("CTAs", len(tr))
for i, name in enumerate(ph):
    v = (tr[:, i] - g0) / 1e3
    v = v[tr[:, i] > 0]
    print(f"{name:10s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us")
