"""Dev: accept kernel time (CUDA graph of 20 calls, preallocated outputs: device time only)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_07223_b200 import accept  # noqa: E402

dev = "cuda"
for V, B, g in ((128256, 1, 4), (128256, 8, 4), (32000, 1, 4)):
    p = torch.softmax(torch.randn((B, g + 1, V), device=dev), -1)
    qd = torch.softmax(torch.randn((B, g, V), device=dev), -1)
    draft = torch.randint(0, V, (B, g), device=dev, dtype=torch.int32)
    u = torch.rand((B, g + 1), device=dev)
    out = (torch.empty(B, dtype=torch.int32, device=dev), torch.empty((B, g + 1), dtype=torch.int32, device=dev))
    for greedy in (False, True):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            accept(p, draft, q=qd, u=u, greedy=greedy, stream=s, out=out)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                for _ in range(20):
                    accept(p, draft, q=qd, u=u, greedy=greedy, stream=s, out=out)
            gr.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            gr.replay()
            e1.record(s)
        torch.cuda.synchronize()
        print(V, B, "greedy" if greedy else "sample", round(e0.elapsed_time(e1) * 1e3 / 20, 2), "us")
