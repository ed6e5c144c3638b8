"""(needs a dev build: make -C paper_2602_07223_b200/csrc EXTRA_NVFLAGS=-DSA_PIPE_TRACE) Dev tool: draft-phase CTA timeline inside the config-2 iteration graph (knob "trace").
  SA_ITER_SKIP=3 python tools/trace_draft.py     # drafts only (selections from an earlier run)
  HQ=32 HKV=4 CTX=131072 K_FIX=9175 LAYERS=8 ...  # config 4's per-GPU shard (4 units of G = 8)
Per draft launch (step, layer): first CTA start, median start, median 'loaded' (after the PDL wait),
median 'computed', max end (us relative to the first draft start)."""
import ctypes
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("SA_AB_ROOT"):  # a dev build from tools/ab_build.sh (e.g. EXTRA_NVFLAGS=-DSA_PIPE_TRACE)
    sys.path.insert(0, os.path.abspath(os.environ["SA_AB_ROOT"]))
import torch  # noqa: E402

from paper_2602_07223_b200 import COLLECT2, Cache, Runner  # noqa: E402
from paper_2602_07223_b200._lib import lib  # noqa: E402

L = int(os.environ.get("LAYERS", 32))
Hq, Hkv, p0, gamma, D = int(os.environ.get("HQ", 32)), int(os.environ.get("HKV", 8)), int(os.environ.get("CTX", 32768)), 4, 128
R = gamma + 1
cache = Cache(L, Hkv, D, p0 + R + 64, page_size=256)
for s in range(0, p0, 2048):
    kk = torch.randn((2048, L * Hkv, D), device="cuda").to(torch.bfloat16)
    cache.append(kk, kk)
KFIX = int(os.environ.get("K_FIX", 0))  # fixed budget k (config 5 sweep points)
r = Runner(cache, Hq, max_rows=R, max_prefix=p0, **({"sparse_ratio": 1e-9, "k_min": KFIX} if KFIX else {}))
r.set_dev_knob("trace", 1)  # dev-only knobs (the library never reads the environment)
for kv in filter(None, os.environ.get("DEV_KNOBS", "").split(",")):  # e.g. DEV_KNOBS=draft_no_pdl=1
    r.set_dev_knob(kv.split("=")[0], int(kv.split("=")[1]))
if os.environ.get("SA_ITER_SKIP"):
    r.set_dev_knob("iter_skip", int(os.environ["SA_ITER_SKIP"]))
r.set_batch([0], [p0])


def rnd(*s):
    return torch.randn(s, device="cuda").to(torch.bfloat16)


qv, kvn, vvn = rnd(L, 1, Hq, R, D), rnd(L, 1, R, Hkv, D), rnd(L, 1, R, Hkv, D)
qd, kdn, vdn = rnd(gamma, L, 1, Hq, D), rnd(gamma, L, 1, Hkv, D), rnd(gamma, L, 1, Hkv, D)
out_v = torch.empty((L, 1, Hq, R, D), device="cuda")
out_d = torch.empty((gamma, L, 1, Hq, D), device="cuda")
for l in range(L):  # selections for every layer (the drafts-only graph reuses them)
    r.verify(l, qv[l], out_v[l], kvn[l], vvn[l])
    r.select(l)
st = torch.cuda.Stream()
args = r.iteration_args(gamma, qv, kvn, vvn, qd, kdn, vdn, out_v, out_d, strategy=COLLECT2, mode=0,
                        scale=1 / math.sqrt(D), use_graph=True)
with torch.cuda.stream(st):
    for _ in range(4):
        r.iteration(args, stream=st)
torch.cuda.synchronize()
path = "/tmp/sa_trace_draft.bin"
assert r.trace_dump(path) == 0
raw = np.fromfile(path, dtype=np.uint64).astype(np.int64)
dr = raw[1024 + 64 * 16384:].reshape(8, 64, 512, 16)
t0 = None
prev = None
print(f"{'step':>4s} {'layer':>5s} {'start':>7s} {'st_max':>7s} | after wait med/max | gathered med/max | computed med/max | end med/max | dt")
for j in range(gamma):
    for l in range(L):
        blk = dr[j, l]
        blk = blk[blk[:, 0] > 0]
        if not len(blk):
            continue
        if t0 is None:
            t0 = blk[:, 0].min()
        v = lambda k: (blk[:, k] - t0) / 1e3  # noqa: E731
        s0, en = v(0), v(4)
        dt = 0.0 if prev is None else en.max() - prev
        prev = en.max()
        if l < 3 or l == L - 1:
            print(f"{j + 1:4d} {l:5d} {s0.min():7.2f} {s0.max():7.2f} | {np.median(v(1)):7.2f} {v(1).max():7.2f} | "
                  f"{np.median(v(2)):7.2f} {v(2).max():7.2f} | {np.median(v(3)):7.2f} {v(3).max():7.2f} | "
                  f"{np.median(en):7.2f} {en.max():7.2f} | {dt:5.2f}  merge: sync1 {np.median(v(8)):7.2f} "
                  f"q_ready {np.median(v(10)):7.2f}/{v(10).max():7.2f} ctamerged {np.median(v(5)):7.2f} "
                  f"pushed {np.median(v(6)):7.2f} inbox {np.median(v(7)):7.2f}/{v(7).max():7.2f}")

# verify phase on the same clock (globaltimer): last layer's end vs the first draft's start
vt = raw[1024:1024 + 64 * 16384].reshape(64, 1024, 16)
v_st = [vt[l][vt[l][:, 0] > 0][:, 0].min() for l in range(L) if (vt[l][:, 0] > 0).any()]
v_en = [vt[l][vt[l][:, 0] > 0][:, 1].max() for l in range(L) if (vt[l][:, 0] > 0).any()]
if v_st:
    d_first = dr[0, 0][dr[0, 0][:, 0] > 0][:, 0].min()
    d_last = max(dr[gamma - 1, l][dr[gamma - 1, l][:, 4] > 0][:, 4].max() for l in range(L) if (dr[gamma - 1, l][:, 4] > 0).any())
    print(f"verify layer0 start -> last verify end {(max(v_en) - min(v_st)) / 1e3:.1f} us; last verify end -> first "
          f"draft start {(d_first - max(v_en)) / 1e3:.1f} us; drafts {(d_last - d_first) / 1e3:.1f} us; "
          f"total {(d_last - min(v_st)) / 1e3:.1f} us")

# per split index: median (over launches) of each CTA's 'computed' and 'gathered' stamps relative to
# its launch's median (which split is the straggler)
CS = int(os.environ.get("CS_HINT", 12))
rel_c, rel_g = {}, {}
for j in range(gamma):
    for l in range(2, L):
        blk = dr[j, l]
        live = np.nonzero(blk[:, 0] > 0)[0]
        if len(live) < CS:
            continue
        med_c, med_g = np.median(blk[live, 3]), np.median(blk[live, 2])
        for c in live:
            s_ = int(c % CS)
            rel_c.setdefault(s_, []).append((blk[c, 3] - med_c) / 1e3)
            rel_g.setdefault(s_, []).append((blk[c, 2] - med_g) / 1e3)
ph = dr[:gamma, 2:L, :, 11:14].reshape(-1, 3)
ph = ph[(ph > 0).all(1) & (ph < 10**6).all(1)]
if len(ph):
    print("warp-0 step<2> cycles (median / p90): QK " + f"{np.median(ph[:, 0]):.0f}/{np.percentile(ph[:, 0], 90):.0f}"
          f"  softmax+P {np.median(ph[:, 1]):.0f}/{np.percentile(ph[:, 1], 90):.0f}"
          f"  PV {np.median(ph[:, 2]):.0f}/{np.percentile(ph[:, 2], 90):.0f}")
print("split: computed-vs-median (us) / gathered-vs-median (us)")
print(" ".join(f"{s_}:{np.median(rel_c[s_]):+.2f}/{np.median(rel_g[s_]):+.2f}" for s_ in sorted(rel_c)))

# stragglers vs SM sharing: for each launch, CTAs that share their SM with another CTA of the SAME
# launch, and their 'computed' lag against the launch median
shared_lag, alone_lag = [], []
for j in range(gamma):
    for l in range(2, L):
        blk = dr[j, l]
        live = np.nonzero(blk[:, 0] > 0)[0]
        if not len(live):
            continue
        sm = blk[live, 15]
        med_c = np.median(blk[live, 3])
        cnt = {s_: int((sm == s_).sum()) for s_ in set(sm.tolist())}
        for c, s_ in zip(live, sm):
            (shared_lag if cnt[s_] > 1 else alone_lag).append((blk[c, 3] - med_c) / 1e3)
if shared_lag or alone_lag:
    print(f"CTAs sharing an SM with a CTA of the same launch: {len(shared_lag)} "
          f"(computed lag median {np.median(shared_lag) if shared_lag else float('nan'):+.2f} us, "
          f"p90 {np.percentile(shared_lag, 90) if shared_lag else float('nan'):+.2f}); alone: {len(alone_lag)} "
          f"(median {np.median(alone_lag):+.2f}, p90 {np.percentile(alone_lag, 90):+.2f})")
