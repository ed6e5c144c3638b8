"""Dev: verify output error vs the reference (oracle/_ref) as a function of the per-CTA accumulation
chain (knob verify_max_splits: 1 = one CTA streams the whole prefix), one sequence, 8 KV heads, G 4.
  python tools/verify_precision.py [p0 ...]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from oracle.pyoracle import Ref, scale_for  # noqa: E402
from paper_2602_07223_b200 import Cache, Runner  # noqa: E402
from tests.helpers import rel_err_elem, rel_err_rows, to_dev_bf16  # noqa: E402

D, Hkv, G, R = 128, 8, 4, 7
Hq = Hkv * G
SCALE = scale_for(D)
ref = Ref()


def bf(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    return ((u + (0x7FFF + ((u >> 16) & 1))) & 0xFFFF0000).view(np.float32)


for p0 in [int(a) for a in sys.argv[1:]] or [16384, 65536]:
    rng = np.random.default_rng(p0)
    K, V = bf(rng.standard_normal((p0, Hkv, D), np.float32)), bf(rng.standard_normal((p0, Hkv, D), np.float32))
    q = bf(rng.standard_normal((1, Hq, R, D), np.float32))
    kn, vn = bf(rng.standard_normal((1, R, Hkv, D), np.float32)), bf(rng.standard_normal((1, R, Hkv, D), np.float32))
    kv = ref.kv(1, Hkv, D, p0 + R + 64)
    for t in range(p0):
        kv.append(K[t], V[t])
    for t in range(R):
        kv.append(kn[0, t], vn[0, t])
    o_ref, _ = kv.verify_layer(0, Hq, q[0], p0, R, SCALE, threads=8)
    for ms in (0, 16, 4, 1):
        c = Cache(1, Hkv, D, p0 + R + 64, page_size=256)
        for c0 in range(0, p0, 8192):
            c.append(torch.from_numpy(K[c0:c0 + 8192]).cuda(), torch.from_numpy(V[c0:c0 + 8192]).cuda())
        r = Runner(c, Hq, max_rows=R, max_prefix=p0)
        if ms:
            r.set_dev_knob("verify_max_splits", ms)
        if os.environ.get("FLUSH"):
            r.set_dev_knob("verify_flush_tiles", int(os.environ["FLUSH"]))
        r.set_batch([0], [p0])
        out = torch.zeros((1, Hq, R, D), dtype=torch.float32, device="cuda")
        r.verify(0, to_dev_bf16(q), out, to_dev_bf16(kn), to_dev_bf16(vn), SCALE)
        got = out.cpu().numpy()[0]
        print(f"p0={p0} flush={os.environ.get('FLUSH', 'default')} max_splits={ms or 'auto'}: rel_err_rows {rel_err_rows(got, o_ref):.3e} "
              f"rel_err_elem {rel_err_elem(got, o_ref):.3e}", flush=True)
        r.close()
        c.close()
