"""Dev probe: does an L2-resident head of the prefix shorten one verify launch?  Config-2 layer shape,
4 layers; layers 1-3 are verified first so layer 0's KV is cold, then (optionally) the first X tokens
of layer 0 (every KV head) are pulled into L2 by sa_kv_read, and layer 0's verify is timed with CUDA
events.  Prints the mean launch time per warm fraction."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2602_07223_b200 import Cache, Runner  # noqa: E402

L, Hq, Hkv, p0, R = 4, 32, 8, 32768, 5
cache = Cache(L, Hkv, 128, p0 + 64, page_size=256)
for s in range(0, p0, 4096):
    kk = torch.randn((4096, L * Hkv, 128), device="cuda").to(torch.bfloat16)
    cache.append(kk, kk)
r = Runner(cache, Hq, max_rows=R, max_prefix=p0)
r.set_batch([0], [p0])
q = torch.randn((1, Hq, R, 128), device="cuda").to(torch.bfloat16)
out = torch.empty((1, Hq, R, 128), device="cuda")
kn = torch.randn((1, R, Hkv, 128), device="cuda").to(torch.bfloat16)
st = torch.cuda.current_stream()
for warm in (0, 2048, 4096, 8192, 0):
    ts = []
    for it in range(12):
        for layer in (1, 2, 3):
            r.verify(layer, q, out, kn, kn)
        if warm:
            for h in range(Hkv):
                cache.read(0, h, 0, warm)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        r.verify(0, q, out, kn, kn)
        e1.record(st)
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"warm tokens {warm:5d} ({100 * warm / p0:4.1f}%): verify {sum(ts) / len(ts):6.2f} us "
          f"(min {min(ts):6.2f})", flush=True)
