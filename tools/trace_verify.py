"""Dev tool: run one config-2 verify layer with SA_TRACE set and print the per-tile pipeline timeline."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SA_TRACE"] = "1"
dump = os.path.join(ROOT, "gpurun_out", "trace.bin")
import torch  # noqa: E402

from paper_2602_07223_b200 import Cache, Runner  # noqa: E402

L, Hq, Hkv, p0, R = 2, 32, 8, 32768, 5
cache = Cache(L, Hkv, 128, p0 + 64, page_size=256)
for s in range(0, p0, 4096):
    kk = torch.randn((4096, L * Hkv, 128), device="cuda").to(torch.bfloat16)
    cache.append(kk, kk)
r = Runner(cache, Hq, max_rows=R, max_prefix=p0)
r.set_batch([0], [p0])
q = torch.randn((1, Hq, R, 128), device="cuda").to(torch.bfloat16)
kn = torch.randn((1, R, Hkv, 128), device="cuda").to(torch.bfloat16)
out = torch.empty((1, Hq, R, 128), device="cuda")
for it in range(3):
    if it == 2:
        os.environ["SA_TRACE_DUMP"] = dump
    r.verify(0, q, out, kn, kn)
torch.cuda.synchronize()
raw = np.fromfile(dump, dtype=np.uint64).astype(np.int64)
ev = raw[:1024].reshape(16, 64)
se = raw[1024:3072].reshape(1024, 2)
se = se[se[:, 0] > 0]
g0 = se[:, 0].min()
st, en = (se[:, 0] - g0) / 1e3, (se[:, 1] - g0) / 1e3
print(f"CTAs {len(se)}: start us min/med/max {st.min():.2f}/{np.median(st):.2f}/{st.max():.2f}; "
      f"end us min/med/max {en.min():.2f}/{np.median(en):.2f}/{en.max():.2f}; dur med {np.median(en - st):.2f}")
order = np.argsort(en)[-6:]
print("slowest CTAs (lin idx, start, end):", [(int(i), round(float(st[i]), 2), round(float(en[i]), 2)) for i in order])
t0 = ev[11, 0]
names = ["K_issued", "V_issued", "QK_issued", "PV_issued", "MMA_kfull", "MMA_vfull", "MMA_pfull", "SM_sfull",
         "SM_pdone", "SM_pempty", "SM_parrive", "start", "SM_ldS", "SM_chk", "SM_bar"]
n = int((ev[2] > 0).sum())
print("tiles", n, "(cycles since start)")
cols = [e for e in range(15) if e != 11]
print("t   " + " ".join(f"{names[e]:>10s}" for e in cols))
for t in range(n):
    print(f"{t:<3d} " + " ".join(f"{(ev[e, t] - t0) if ev[e, t] else -1:10d}" for e in cols))
