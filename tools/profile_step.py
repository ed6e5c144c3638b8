"""Profiling driver: config-2-shaped iterations (fewer layers by default) launched without a graph
so ncu sees every kernel.  Usage (on the GPU box):
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python tools/profile_step.py --layers 4 --iters 2
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--gamma", type=int, default=4)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--graph", action="store_true")
    ap.add_argument("--mode", type=int, default=0)
    a = ap.parse_args()
    import torch

    from paper_2602_07223_b200 import COLLECT2, Cache, Runner
    L, Hq, Hkv, p0, gamma, B, D = a.layers, a.hq, a.hkv, a.ctx, a.gamma, a.batch, 128
    R = gamma + 1
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    cache = Cache(L, Hkv, D, p0 + R + 64, max_seqs=B)
    for b in range(B):
        done = 0
        while done < p0:
            n = min(4096, p0 - done)
            kk = torch.randn((n, L * Hkv, D), generator=g, device="cuda").to(torch.bfloat16)
            cache.append(kk, kk, seq=b)
            done += n
    r = Runner(cache, Hq, max_rows=R, max_prefix=p0, max_batch=B, sparse_ratio=0.07, k_min=16)
    r.set_batch(list(range(B)), [p0] * B)

    def rnd(*s):
        return torch.randn(s, generator=g, device="cuda").to(torch.bfloat16)

    qv, kvn, vvn = rnd(L, B, Hq, R, D), rnd(L, B, R, Hkv, D), rnd(L, B, R, Hkv, D)
    qd, kdn, vdn = rnd(gamma, L, B, Hq, D), rnd(gamma, L, B, Hkv, D), rnd(gamma, L, B, Hkv, D)
    out_v = torch.empty((L, B, Hq, R, D), device="cuda")
    out_d = torch.empty((gamma, L, B, Hq, D), device="cuda")
    s = torch.cuda.Stream()
    args = r.iteration_args(gamma, qv, kvn, vvn, qd, kdn, vdn, out_v, out_d, strategy=COLLECT2, mode=a.mode,
                            scale=1 / math.sqrt(D), use_graph=a.graph)
    with torch.cuda.stream(s):
        for _ in range(a.iters):
            r.iteration(args, stream=s)
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
