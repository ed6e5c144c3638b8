"""Dev probe: can one e2e step (upload of step i+1, the iteration of step i through sa_iteration_run, the
read-back of step i-1) be captured into ONE CUDA graph per buffer set, so consecutive steps are
back-to-back graph launches on one stream (no cross-stream event waits between them)?  Config 2 shape.
Prints ms/step for: compute only, the event-pipelined e2e (bench.py's scheme), and the graph scheme."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2602_07223_b200 import COLLECT2, Cache, Runner  # noqa: E402

L, Hq, Hkv, p0, gamma, D = 32, 32, 8, 32768, 4, 128
R, NS = gamma + 1, 3
cache = Cache(L, Hkv, D, p0 + R + 64, page_size=256)
for s in range(0, p0, 2048):
    kk = torch.randn((2048, L * Hkv, D), device="cuda").to(torch.bfloat16)
    cache.append(kk, kk)
r = Runner(cache, Hq, max_rows=R, max_prefix=p0)
r.set_batch([0], [p0])


def rnd(*s):
    return torch.randn(s, device="cuda").to(torch.bfloat16)


sets = []
for _ in range(NS):
    t = [rnd(L, 1, Hq, R, D), rnd(L, 1, R, Hkv, D), rnd(L, 1, R, Hkv, D), rnd(gamma, L, 1, Hq, D),
         rnd(gamma, L, 1, Hkv, D), rnd(gamma, L, 1, Hkv, D), torch.empty((L, 1, Hq, R, D), device="cuda"),
         torch.empty((gamma, L, 1, Hq, D), device="cuda")]
    sets.append((t, r.iteration_args(gamma, *t[:6], t[6], t[7], strategy=COLLECT2, scale=1 / math.sqrt(D)),
                 r.iteration_args(gamma, *t[:6], t[6], t[7], strategy=COLLECT2, scale=1 / math.sqrt(D),
                                  use_graph=False)))  # direct enqueue: captured by the outer graph
hin = [[x.cpu().pin_memory() for x in st[0][:6]] for st in sets]
hout = [[torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in st[0][6:]] for st in sets]
main = torch.cuda.Stream()


def timed(fn, n=20):
    for i in range(NS + 1):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for i in range(n):
        fn(i)
    b.record(main)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


print(f"compute only {timed(lambda i: r.iteration(sets[i % NS][1], stream=main)):.4f} ms/step", flush=True)

# one graph per set j: step i (set j = i % NS) computes set j, uploads set (j+1) % NS, reads back set (j-1) % NS
graphs = []
up, down = torch.cuda.Stream(), torch.cuda.Stream()
try:
    for j in range(NS):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=main):
            cur = torch.cuda.current_stream()
            fork = torch.cuda.Event()
            fork.record(cur)
            up.wait_event(fork)
            down.wait_event(fork)
            with torch.cuda.stream(up):
                for h, d in zip(hin[(j + 1) % NS], sets[(j + 1) % NS][0][:6]):
                    d.copy_(h, non_blocking=True)
            with torch.cuda.stream(down):
                for h, d in zip(hout[(j - 1) % NS], sets[(j - 1) % NS][0][6:]):
                    h.copy_(d, non_blocking=True)
            r.iteration(sets[j][2], stream=cur)
            e_up, e_down = torch.cuda.Event(), torch.cuda.Event()
            e_up.record(up)
            e_down.record(down)
            cur.wait_event(e_up)
            cur.wait_event(e_down)
        graphs.append(g)
    with torch.cuda.stream(main):
        print(f"graph e2e {timed(lambda i: graphs[i % NS].replay()):.4f} ms/step", flush=True)
except Exception as e:  # noqa: BLE001
    print("graph capture failed:", repr(e)[:300], flush=True)
