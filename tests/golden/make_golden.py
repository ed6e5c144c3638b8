"""Generate tests/golden/golden_v1.npz by running the REFERENCE's own code (oracle/_ref, i.e.
/root/reference/proj/src/{attention,selection,kv_store}.cpp compiled against oracle/shim/Eigen)
on seeded CounterRng inputs.  Run in the build container (needs /root/reference):

    make -C oracle && python tests/golden/make_golden.py

The GPU box never reads /root/reference; tests compare against this committed file.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.counter_rng import normal_bf16  # noqa: E402
from oracle.pyoracle import ALL_DRAFT, COLLECT2, COLLECT2_WEIGHTS, LAST_ACCEPTED, Ref, scale_for  # noqa: E402


def main():
    ref = Ref()
    d = 128
    s = scale_for(d)
    g = {"scale": np.float32(s)}
    # attend_collect
    g["ac_q"] = normal_bf16(101, 1, (d,))
    g["ac_Kp"], g["ac_Vp"] = normal_bf16(101, 2, (45, d)), normal_bf16(101, 3, (45, d))
    g["ac_Kw"], g["ac_Vw"] = normal_bf16(101, 4, (3, d)), normal_bf16(101, 5, (3, d))
    g["ac_out"], g["ac_logits"] = ref.attend_collect(g["ac_q"], g["ac_Kp"], g["ac_Vp"], g["ac_Kw"], g["ac_Vw"], s)
    # selection strategies on one LogitMatrix (4 heads x 5 rows x 80 cols)
    g["sel_L"] = normal_bf16(102, 1, (4, 5, 80), scale=8.0)
    for i, strat in enumerate((ALL_DRAFT, COLLECT2, COLLECT2_WEIGHTS, LAST_ACCEPTED)):
        idx = ref.select(strat, g["sel_L"], [1, 2, 3, 4, 5], 0.25, 4, accepted=2)
        g[f"sel_{i}"] = np.pad(idx, (0, 80 - len(idx)))
        g[f"sel_{i}_n"] = np.int64(len(idx))
    # verify + draft compositions over a reference KvStore (2 layers, 2 KV heads, 8 q heads)
    L, Hkv, Hq, p0, R = 2, 2, 8, 150, 3
    g["vl_shape"] = np.array([L, Hkv, d])
    g["vl_p0"], g["vl_R"], g["vl_Hq"] = np.int64(p0), np.int64(R), np.int64(Hq)
    g["vl_K"] = normal_bf16(103, 1, (p0 + R, L * Hkv, d))
    g["vl_V"] = normal_bf16(103, 2, (p0 + R, L * Hkv, d))
    g["vl_q"] = normal_bf16(103, 3, (Hq, R, d))
    g["dr_q"] = normal_bf16(103, 4, (Hq, d))
    kv = ref.kv(L, Hkv, d, 512)
    for t in range(p0 + R):
        kv.append(g["vl_K"][t], g["vl_V"][t])
    for layer in range(L):
        g[f"vl_out_{layer}"], g[f"vl_logits_{layer}"] = kv.verify_layer(layer, Hq, g["vl_q"], p0, R, s)
        sets = []
        for h in range(Hkv):
            sel = np.sort(np.random.default_rng(1000 + 10 * layer + h).choice(p0, 20, replace=False)).astype(np.int64)
            g[f"dr_set_{layer}_{h}"] = sel
            sets.append(sel)
        g[f"dr_out_{layer}"] = kv.draft_layer(layer, Hq, g["dr_q"], sets, p0, 2, s)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_v1.npz")
    np.savez_compressed(out, **g)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
