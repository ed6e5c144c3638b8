"""Dev probe: where the e2e leg's extra time goes (compute alone, + uploads, + read-backs)."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2602_07223_b200 import COLLECT2, Cache, Runner  # noqa: E402

L, Hq, Hkv, p0, gamma, D = 32, 32, 8, 32768, 4, 128
R = gamma + 1
cache = Cache(L, Hkv, D, p0 + R + 64, page_size=256)
for s in range(0, p0, 2048):
    kk = torch.randn((2048, L * Hkv, D), device="cuda").to(torch.bfloat16)
    cache.append(kk, kk)
r = Runner(cache, Hq, max_rows=R, max_prefix=p0)
r.set_batch([0], [p0])


def rnd(*s):
    return torch.randn(s, device="cuda").to(torch.bfloat16)


sets = []
for _ in range(2):
    t = [rnd(L, 1, Hq, R, D), rnd(L, 1, R, Hkv, D), rnd(L, 1, R, Hkv, D), rnd(gamma, L, 1, Hq, D),
         rnd(gamma, L, 1, Hkv, D), rnd(gamma, L, 1, Hkv, D), torch.empty((L, 1, Hq, R, D), device="cuda"),
         torch.empty((gamma, L, 1, Hq, D), device="cuda")]
    sets.append((t, r.iteration_args(gamma, *t[:6], t[6], t[7], strategy=COLLECT2, scale=1 / math.sqrt(D))))
hin = [[x.cpu().pin_memory() for x in st[0][:6]] for st in sets]
hout = [[torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in st[0][6:]] for st in sets]
main, up, down = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def run(n, do_up, do_down):
    evs = []
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for i in range(n):
        st = i % 2
        if do_up:
            with torch.cuda.stream(up):
                for h, d in zip(hin[st], sets[st][0][:6]):
                    d.copy_(h, non_blocking=True)
            e = torch.cuda.Event()
            e.record(up)
            main.wait_event(e)
        r.iteration(sets[st][1], stream=main)
        if do_down:
            e2 = torch.cuda.Event()
            e2.record(main)
            down.wait_event(e2)
            with torch.cuda.stream(down):
                for h, d in zip(hout[st], sets[st][0][6:]):
                    h.copy_(d, non_blocking=True)
            evs.append(e2)
    b.record(main)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for _ in range(2):
    run(4, True, True)
for mode in [(False, False), (True, False), (False, True), (True, True)]:
    print(mode, f"{run(20, *mode):.4f} ms/step")
# copy-only timings
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(up)
for _ in range(20):
    with torch.cuda.stream(up):
        for h, d in zip(hin[0], sets[0][0][:6]):
            d.copy_(h, non_blocking=True)
b.record(up)
torch.cuda.synchronize()
print(f"H2D alone {a.elapsed_time(b) / 20:.4f} ms")
a.record(down)
for _ in range(20):
    with torch.cuda.stream(down):
        for h, d in zip(hout[0], sets[0][0][6:]):
            h.copy_(d, non_blocking=True)
b.record(down)
torch.cuda.synchronize()
print(f"D2H alone {a.elapsed_time(b) / 20:.4f} ms")
