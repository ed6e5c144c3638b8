"""Dev tool: config-2 verify of one layer with the "trace" knob set, after 3 other layers have streamed
through L2 (so the traced layer is read from DRAM): CTA start / main-loop end / end and the per-tile
pipeline timeline of CTA 0.  The per-tile stamps need a dev build of the library:
  make -C paper_2602_07223_b200/csrc EXTRA_NVFLAGS=-DSA_PIPE_TRACE   (the product build compiles them out)"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2602_07223_b200 import Cache, Runner  # noqa: E402
from paper_2602_07223_b200._lib import lib  # noqa: E402

L, Hq, Hkv, p0, R = 4, 32, 8, int(os.environ.get("CTX", 32768)), 5
cache = Cache(L, Hkv, 128, p0 + 64, page_size=256)
for s in range(0, p0, 4096):
    kk = torch.randn((4096, L * Hkv, 128), device="cuda").to(torch.bfloat16)
    cache.append(kk, kk)
r = Runner(cache, Hq, max_rows=R, max_prefix=p0)
r.set_dev_knob("trace", 1)  # dev-only knobs (the library never reads the environment)
if os.environ.get("SA_ITER_SKIP"):
    r.set_dev_knob("iter_skip", int(os.environ["SA_ITER_SKIP"]))
r.set_batch([0], [p0])
q = torch.randn((1, Hq, R, 128), device="cuda").to(torch.bfloat16)
kn = torch.randn((1, R, Hkv, 128), device="cuda").to(torch.bfloat16)
out = torch.empty((1, Hq, R, 128), device="cuda")
for it in range(2):
    for layer in (1, 2, 3, 0):
        r.verify(layer, q, out, kn, kn, score_layout=1)
torch.cuda.synchronize()
dump = "/tmp/sa_trace_verify.bin"

assert r.trace_dump(dump) == 0
raw = np.fromfile(dump, dtype=np.uint64).astype(np.int64)
ev = raw[:1024].reshape(16, 64)
se = raw[1024:1024 + 16384].reshape(1024, 16)
se = se[se[:, 0] > 0]
g0 = se[:, 0].min()
rel = lambda k: (se[:, k] - g0) / 1e3  # noqa: E731
st, en, ml, pv, sto, cnt, mrg = rel(0), rel(1), rel(2), rel(4), rel(5), rel(6), rel(7)
tiles, split = se[:, 3] & 0xFFFFFFFF, se[:, 3] >> 32
print(f"CTAs {len(se)}: start us min/med/max {st.min():.2f}/{np.median(st):.2f}/{st.max():.2f}; "
      f"main-loop end min/med/max {ml.min():.2f}/{np.median(ml):.2f}/{ml.max():.2f}; "
      f"end min/med/max {en.min():.2f}/{np.median(en):.2f}/{en.max():.2f}")
has = se[:, 5] > 0
print(f"epilogue detail (us): pv_done->both_wg {np.median((rel(10) - pv)[has]):.2f}  ->fin_l {np.median((rel(11) - rel(10))[has]):.2f}  "
      f"->O_stored {np.median((rel(12) - rel(11))[has]):.2f}  ->barrier {np.median((sto - rel(12))[has]):.2f}")
print(f"epilogue medians (us): loop_end->pv_done {np.median(pv - ml):.2f}  pv_done->partial_stored "
      f"{np.median((sto - pv)[has]):.2f}  stored->counted {np.median((cnt - sto)[has]):.2f}  counted->end(non-merger) "
      f"{np.median((en - cnt)[has]):.2f}")
mg = se[:, 12] > 0
if mg.any():
    print(f"merger detail (us): counted->landed {np.median((rel(12) - cnt)[mg]):.2f}  weights {np.median((rel(13) - rel(12))[mg]):.2f}  "
          f"barrier {np.median((rel(14) - rel(13))[mg]):.2f}  combine {np.median((rel(15) - rel(14))[mg]):.2f}  "
          f"->end {np.median((en - rel(15))[mg]):.2f}")
mg = se[:, 7] > 0
if mg.any():
    w8, c9 = rel(8), rel(9)
    print(f"mergers {mg.sum()}: counted->inputs_landed med {np.median((mrg - cnt)[mg]):.2f}  landed->weights "
          f"{np.median((w8 - mrg)[mg]):.2f}  weights->combined {np.median((c9 - w8)[mg]):.2f}  combined->end "
          f"{np.median((en - c9)[mg]):.2f}  merger end max {en[mg].max():.2f}")
order = np.argsort(en)[-8:]
print("slowest CTAs (lin, split, wg0 tiles, start, loop_end, end):",
      [(int(i), int(split[i]), int(tiles[i]), round(float(st[i]), 2), round(float(ml[i]), 2), round(float(en[i]), 2)) for i in order])
print("wg0 tiles per CTA: min/med/max", tiles.min(), np.median(tiles), tiles.max())
t0 = ev[11, 0]
names = ["K_issued", "V_issued", "QK_issued", "PV_issued", "MMA_kfull", "MMA_vfull", "MMA_pfull", "SM_sfull",
         "SM_pdone", "SM_pempty", "SM_parrive", "start", "SM_ldS", "SM_chk", "SM_bar"]
n = int((ev[2] > 0).sum())
print("tiles", n, "(cycles since start)")
cols = [e for e in range(15) if e != 11]
print("t   " + " ".join(f"{names[e]:>10s}" for e in cols))
for t in range(n):
    print(f"{t:<3d} " + " ".join(f"{(ev[e, t] - t0) if ev[e, t] else -1:10d}" for e in cols))
