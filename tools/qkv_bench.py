import os
"""Producer timing: L chained projections (graph, PDL) at the Llama-3.1-8B shape; prints JSON."""
import json
import sys

import torch

from paper_2602_07223_b200 import QkvProjection


def main():
    L, D, Hq, Hkv = 32, 4096, 32, 8
    n_out = (Hq + 2 * Hkv) * 128
    w = (torch.randn(L, n_out, D, device="cuda") / 64).to(torch.bfloat16)
    gain = torch.ones(L, D, device="cuda")
    proj = QkvProjection(w, gain, Hq, Hkv)
    if os.environ.get("SA_QKV_DEV"):  # tool parameter -> dev knob
        proj.set_dev_knob("dev", int(os.environ["SA_QKV_DEV"]))
    out = {}
    for B, rows in ((1, 5), (1, 1), (4, 5), (16, 5)):
        x = torch.randn(B, rows, D, device="cuda")
        pos = torch.full((B,), 32768, dtype=torch.int32, device="cuda")
        q = torch.empty(B, Hq, rows, 128, dtype=torch.bfloat16, device="cuda")
        k = torch.empty(B, rows, Hkv, 128, dtype=torch.bfloat16, device="cuda")
        v = torch.empty_like(k)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for l in range(L):
                proj.project(l, x, pos, q, k, v, stream=s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for l in range(L):
                    proj.project(l, x, pos, q, k, v, stream=s)
            for _ in range(5):
                g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 20
            e0.record(s)
            for _ in range(n):
                g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (n * L)
        nbytes = n_out * D * 2 + B * rows * (D * 4 + n_out * 2)
        out[f"B{B}xR{rows}"] = {"us_per_layer": round(us, 2), "gbs": round(nbytes / us / 1e3, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
