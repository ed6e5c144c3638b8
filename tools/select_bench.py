"""Dev: select kernel time with its scores L2-resident (config-2 layer: 8 KV heads, G 4, 32K columns).
Per-KV-head mode (fp32 sums, not consumed) so the same scores are selected repeatedly; per-layer mode
re-runs one verify before every select (the int64 slot is zeroed as it is consumed) and reports
select time = (verify + select) - verify.  Both kernels: the cluster select and select_legacy."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2602_07223_b200 import Cache, Runner  # noqa: E402

L, Hq, Hkv, R = 1, 32, 8, 5
p0 = int(os.environ.get("CTX", 32768))
cache = Cache(L, Hkv, 128, p0 + 64, page_size=256)
for s in range(0, p0, 4096):
    kk = torch.randn((min(4096, p0 - s), L * Hkv, 128), device="cuda").to(torch.bfloat16)
    cache.append(kk, kk)
q = torch.randn((1, Hq, R, 128), device="cuda").to(torch.bfloat16)
kn = torch.randn((1, R, Hkv, 128), device="cuda").to(torch.bfloat16)
out = torch.empty((1, Hq, R, 128), device="cuda")
st = torch.cuda.current_stream()


def timed(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(n):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


for legacy in (1, 0):
    r = Runner(cache, Hq, max_rows=R, max_prefix=p0)
    r.set_dev_knob("select_legacy", legacy)
    r.set_batch([0], [p0])
    cache.set_size(p0)
    r.verify(0, q, out, kn, kn, score_layout=1)
    t_kv = timed(lambda: r.select(0, mode=1))
    cache.set_size(p0)
    t_v = timed(lambda: (cache.set_size(p0), r.verify(0, q, out, kn, kn, score_layout=0)))
    t_vs = timed(lambda: (cache.set_size(p0), r.verify(0, q, out, kn, kn, score_layout=0), r.select(0, mode=0)))
    print(f"{'legacy (1 CTA)' if legacy else 'cluster (8 CTAs)'}: per-KV-head select (8 sets) {t_kv:6.2f} us; "
          f"per-layer select {t_vs - t_v:6.2f} us (verify {t_v:.2f}, verify+select {t_vs:.2f})", flush=True)
    r.close()
