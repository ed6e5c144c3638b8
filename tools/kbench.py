"""Dev tool: CUDA-event timing of each hot-path kernel in isolation (config-2 shapes, warm, back to
back on one stream) — complements ncu's serialised launch list."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2602_07223_b200 import Cache, Runner  # noqa: E402


def timed(fn, n=50, warm=5):
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(n):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3  # us


def main():
    L, Hq, Hkv, p0, gamma = 4, 32, 8, int(os.environ.get("CTX", 32768)), 4
    R, D = gamma + 1, 128
    cache = Cache(L, Hkv, D, p0 + 64, page_size=256)
    for s in range(0, p0, 4096):
        kk = torch.randn((min(4096, p0 - s), L * Hkv, D), device="cuda").to(torch.bfloat16)
        cache.append(kk, kk)
    r = Runner(cache, Hq, max_rows=R, max_prefix=p0)
    r.set_batch([0], [p0])
    q = torch.randn((1, Hq, R, D), device="cuda").to(torch.bfloat16)
    kn = torch.randn((1, R, Hkv, D), device="cuda").to(torch.bfloat16)
    out = torch.empty((1, Hq, R, D), device="cuda")
    sc = 1 / math.sqrt(D)
    layer = [0]

    def verify():
        layer[0] = (layer[0] + 1) % L
        r.verify(layer[0], q, out, kn, kn, sc, score_layout=1)

    tv = timed(verify)
    tsel_kv = timed(lambda: r.select(1, mode=1))

    def sel_layer():
        r.verify(1, q, out, kn, kn, sc)
        r.select(1)

    tvs = timed(sel_layer)
    tsel = tvs - tv
    qd = torch.randn((1, Hq, D), device="cuda").to(torch.bfloat16)
    kd = torch.randn((1, Hkv, D), device="cuda").to(torch.bfloat16)
    od = torch.empty((1, Hq, D), device="cuda")

    def draft():
        layer[0] = (layer[0] + 1) % L
        r.draft(layer[0], 2, qd, od, kd, kd)

    td = timed(draft)
    kv_bytes = p0 * Hkv * 512
    k = r.selection(1, 1)[1][0, 0]
    print(f"verify  {tv:8.2f} us  {kv_bytes / tv / 1e3:8.1f} GB/s (KV only)")
    print(f"select  {tsel:8.2f} us (per layer, = verify+select - verify)   per-KV-head select {tsel_kv:8.2f} us")
    print(f"draft   {td:8.2f} us  k={k}  {(k + 2) * Hkv * 512 / td / 1e3:8.1f} GB/s")


if __name__ == "__main__":
    main()
