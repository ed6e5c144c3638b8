"""GPU parity: every op through the C ABI vs the reference's own CPU code (oracle/_ref) on the
same seeded bf16-representable inputs.  Bars (north star / SURVEY.md §8c):
  attention outputs  <= 2e-3 max relative error (we also assert the much tighter measured level)
  logits             |d| <= 1e-5 * sum_j |q_j k_j|
  index sets         bit-exact outside the 2e-3 score tie band; exact on planted exact ties
"""
import numpy as np
import pytest

from oracle.counter_rng import normal_bf16
from oracle.pyoracle import ALL_DRAFT, COLLECT2, LAST_ACCEPTED, scale_for

from .helpers import D, Matched, check_selection, rel_err_elem, rel_err_rows, to_dev_bf16

pytestmark = pytest.mark.gpu
SCALE = scale_for(D)


def _lib():
    from paper_2602_07223_b200 import Runner, SpecAttnError, selection_k
    return Runner, SpecAttnError, selection_k


# ----------------------------------------------------------------------------------- KV cache

def test_cache_append_read_gather_truncate(cuda, ref):
    torch = cuda
    _, SpecAttnError, _ = _lib()
    m = Matched(ref, L=2, Hkv=2, n_tokens=300, seed=11, max_context=400, page_size=128)
    c, kv = m.cache, m.refs[0]
    assert c.size() == kv.size() == 300
    for layer in range(2):
        for h in range(2):
            K, V = c.read(layer, h, 0, 300)
            Kr, Vr = kv.rows(layer, h, 0, 300)
            assert np.array_equal(K.cpu().numpy(), Kr) and np.array_equal(V.cpu().numpy(), Vr)
    idx = [0, 5, 63, 64, 65, 200, 299]
    K, V = c.gather(1, 1, idx)
    Kr, Vr = kv.gather(1, 1, idx)
    assert np.array_equal(K.cpu().numpy(), Kr) and np.array_equal(V.cpu().numpy(), Vr)
    # rollback semantics: truncate then append overwrites
    c.set_committed(250)
    kv.set_committed(250)
    c.truncate(120)
    kv.truncate(120)
    assert c.committed() == kv.committed() == 120
    newk = normal_bf16(12, 1, (1, 4, D))
    newv = normal_bf16(12, 2, (1, 4, D))
    c.append(torch.from_numpy(newk).cuda(), torch.from_numpy(newv).cuda())
    kv.append(newk[0], newv[0])
    K, _ = c.read(0, 1, 118, 3)
    Kr, _ = kv.rows(0, 1, 118, 3)
    assert np.array_equal(K.cpu().numpy(), Kr)
    # error taxonomy
    with pytest.raises(SpecAttnError) as e:
        c.truncate(500)
    assert e.value.status == "out_of_range"
    with pytest.raises(SpecAttnError) as e:
        c.gather(0, 0, [3, 2])
    assert e.value.status == "out_of_range"
    with pytest.raises(SpecAttnError) as e:
        c.gather(0, 0, [121])
    assert e.value.status == "out_of_range"
    big = torch.zeros((400, 4, D), dtype=torch.float32, device="cuda")
    with pytest.raises(SpecAttnError) as e:
        c.append(big, big)
    assert e.value.status == "length_error"
    assert c.bytes_per_token() == (2 * 2 * 2 * D * 4, 2 * 2 * 2 * D * 2)
    # fp32 input that is not bf16-representable rounds to nearest even (documented deviation)
    x = torch.full((1, 4, D), 1.0 + 2.0 ** -10, dtype=torch.float32, device="cuda")
    c.append(x, x)
    K, _ = c.read(0, 0, c.size() - 1, 1)
    assert float(K[0, 0]) == 1.0


# ----------------------------------------------------------------------------------- verify

VERIFY_CASES = [
    # (Hkv, G, R, p0s, page)   — covers MT = 1..4, ragged / tiny / empty prefixes, batching
    (8, 4, 5, [4096], 256),      # config 1 (G*R = 20 -> MT 2)
    (2, 4, 7, [1000], 128),       # gamma 6 (config 3 shape), ragged p0
    (2, 8, 5, [777], 128),       # 70B group (G = 8) -> MT 3
    (1, 8, 7, [300], 128),        # G*R + 2 = 58 -> MT 4
    (2, 1, 2, [130], 128),        # MT 1
    (2, 4, 5, [0, 50, 2049], 128),  # empty prefix, < one tile, multi-sequence batch
]


def _run_verify(ref, Hkv, G, R, p0s, page, seed=31, collect_all=True, score_layout=1):
    import torch
    Runner, _, _ = _lib()
    Hq = Hkv * G
    B = len(p0s)
    m = Matched(ref, L=2, Hkv=Hkv, n_tokens=0, seed=seed, max_context=max(p0s) + R + 64, page_size=page,
                n_seqs=B, lens=p0s)
    r = Runner(m.cache, Hq, max_rows=R, max_prefix=max(p0s), max_batch=B)
    r.set_batch(list(range(B)), p0s)
    layer = 1
    q = normal_bf16(seed, 10, (B, Hq, R, D))
    kn = normal_bf16(seed, 11, (B, R, Hkv, D))
    vn = normal_bf16(seed, 12, (B, R, Hkv, D))
    out = torch.zeros((B, Hq, R, D), dtype=torch.float32, device="cuda")
    ld = max(64, max(p0s))
    logits = torch.full((B, Hq, R, ld), float("nan"), dtype=torch.float32, device="cuda")
    mask = (1 | (1 << (R - 1)))
    r.verify(layer, to_dev_bf16(q), out, to_dev_bf16(kn), to_dev_bf16(vn), SCALE, score_row_mask=mask,
             logits=logits, collect_row_mask=(1 << R) - 1, score_layout=score_layout)
    torch.cuda.synchronize()
    if score_layout == 1:  # per-KV-head fp32 column sums
        sp, sld = r.scores(layer)
        from paper_2602_07223_b200._lib import _device_bytes
        scores = _device_bytes(sp, B * Hkv * sld * 4).view(torch.float32).reshape(B, Hkv, sld).cpu().numpy()
    else:  # per-layer fixed-point sums over all KV heads (2^-32 units)
        scores = r.layer_scores(layer)
    res = []
    for b in range(B):
        kv = m.refs[b]
        # the reference appends the gamma+1 verify tokens for all layers
        for t in range(R):
            kk = normal_bf16(seed + 99, t, (2 * Hkv, D))
            vv = normal_bf16(seed + 98, t, (2 * Hkv, D))
            kk[Hkv:] = kn[b, t]
            vv[Hkv:] = vn[b, t]
            kv.append(kk, vv)
        o_ref, l_ref = kv.verify_layer(layer, Hq, q[b], p0s[b], R, SCALE, threads=8)
        res.append((o_ref, l_ref))
    return m, r, q, kn, vn, out.cpu().numpy(), logits.cpu().numpy(), scores, res


@pytest.mark.parametrize("Hkv,G,R,p0s,page", VERIFY_CASES)
def test_verify_parity(cuda, ref, Hkv, G, R, p0s, page):
    torch = cuda
    m, r, q, kn, vn, out, logits, scores, res = _run_verify(ref, Hkv, G, R, p0s, page)
    Hq = Hkv * G
    for b, p0 in enumerate(p0s):
        o_ref, l_ref = res[b]
        assert rel_err_rows(out[b], o_ref) < 2e-4, rel_err_rows(out[b], o_ref)
        assert rel_err_elem(out[b], o_ref) < 2e-3
        if p0:
            # logits byproduct: |d| <= 1e-5 * sum_j |q_j k_j|
            Kh = m.K[b][:p0].reshape(p0, 2, Hkv, D)[:, 1]  # layer 1
            g_of_h = np.arange(Hq) // G
            bound = np.einsum("hrd,phd->hrp", np.abs(q[b]), np.abs(Kh[:, g_of_h]))
            assert np.all(np.abs(logits[b][:, :, :p0] - l_ref) <= 1e-5 * bound + 1e-30)
            # fused Collect-2 score byproduct == score_columns over rows {1, R} (per KV head sums)
            rows = sorted({0, R - 1})
            want = l_ref[:, rows, :].astype(np.float64).reshape(Hkv, G * len(rows), p0).sum(1)
            tol = 2e-5 * bound[:, rows, :].reshape(Hkv, G * len(rows), p0).sum(1) + 1e-4
            assert np.all(np.abs(scores[b][:, :p0] - want) <= tol)
        # fused append: window rows landed in the cache
        K, V = m.cache.read(1, Hkv - 1, p0, R, seq=b) if m.cache.size(b) >= p0 + R else (None, None)
        if K is None:
            m.cache.set_size(p0 + R, seq=b)
            K, V = m.cache.read(1, Hkv - 1, p0, R, seq=b)
        assert np.array_equal(K.cpu().numpy(), kn[b, :, Hkv - 1]) and np.array_equal(V.cpu().numpy(), vn[b, :, Hkv - 1])
    torch.cuda.synchronize()


# per-layer scores (score_layout 0) take the row-split kernel at MMA width N >= 48: balanced row pairs at
# N = 48 (20 / 20, 18 / 18, 22 / 22 rows), 8-row chunks at N = 64 (32 / 24); outputs, raw logits and the
# int64 Collect-2 column sums vs the reference
@pytest.mark.parametrize("Hkv,G,R,p0s", [(2, 8, 5, [777]), (1, 4, 9, [1500]), (2, 4, 11, [900, 64]), (1, 8, 7, [300])])
def test_verify_row_split_parity(cuda, ref, Hkv, G, R, p0s):
    m, r, q, kn, vn, out, logits, fx, res = _run_verify(ref, Hkv, G, R, p0s, 128, seed=47, score_layout=0)
    Hq = Hkv * G
    for b, p0 in enumerate(p0s):
        o_ref, l_ref = res[b]
        assert rel_err_rows(out[b], o_ref) < 2e-4, rel_err_rows(out[b], o_ref)
        assert rel_err_elem(out[b], o_ref) < 2e-3
        if p0:
            Kh = m.K[b][:p0].reshape(p0, 2, Hkv, D)[:, 1]
            bound = np.einsum("hrd,phd->hrp", np.abs(q[b]), np.abs(Kh[:, np.arange(Hq) // G]))
            assert np.all(np.abs(logits[b][:, :, :p0] - l_ref) <= 1e-5 * bound + 1e-30)
            rows = [0, R - 1]
            want = l_ref[:, rows, :].astype(np.float64).sum((0, 1))
            got = fx[b, :p0].astype(np.float64) / 2.0 ** 32
            assert np.all(np.abs(got - want) <= 2e-5 * bound[:, rows].sum((0, 1)) + 1e-4)


def test_layer_scores_fixed_point(cuda, ref):
    """Per-layer score byproduct: int64 column sums over ALL KV heads (fixed point, 2^-32) ==
    score_columns' numerator (selection.cpp:93-106); consumed (zeroed) by the per-layer select."""
    Hkv, G, R, p0 = 4, 4, 5, 3000
    m, r, q, kn, vn, out, logits, fx, res = _run_verify(ref, Hkv, G, R, [p0], 128, seed=45, score_layout=0)
    l_ref = res[0][1]
    rows = [0, R - 1]
    want = l_ref[:, rows, :].astype(np.float64).sum((0, 1))
    got = fx[0, :p0].astype(np.float64) / 2.0 ** 32
    Kh = m.K[0][:p0].reshape(p0, 2, Hkv, D)[:, 1]
    bound = np.einsum("hrd,phd->hrp", np.abs(q[0]), np.abs(Kh[:, np.arange(Hkv * G) // G]))[:, rows].sum((0, 1))
    assert np.all(np.abs(got - want) <= 2e-5 * bound + 1e-4)
    assert not fx[0, p0:].any()
    r.select(1, mode=0, rows_in_score=2)
    assert not r.layer_scores(1).any()  # re-armed for the next verify
    # a second verify on the same slot without a select in between must not double-accumulate
    import torch
    out2 = torch.zeros((1, Hkv * G, R, D), dtype=torch.float32, device="cuda")
    for _ in range(2):
        r.verify(1, to_dev_bf16(q), out2, to_dev_bf16(kn), to_dev_bf16(vn), SCALE, score_row_mask=1 | (1 << (R - 1)))
    assert np.array_equal(r.layer_scores(1), fx)


def test_verify_deterministic(cuda, ref):
    for layout in (0, 1):
        a = _run_verify(ref, 2, 4, 5, [1500], 128, seed=41, score_layout=layout)
        b = _run_verify(ref, 2, 4, 5, [1500], 128, seed=41, score_layout=layout)
        assert np.array_equal(a[5], b[5]) and np.array_equal(a[7], b[7])


# ----------------------------------------------------------------------------------- select

def _gpu_select(r, slot, mode, n_sets, rows_in_score):
    r.select(slot, mode=mode, rows_in_score=rows_in_score)
    idx, cnt = r.selection(slot, n_sets)
    return idx, cnt


@pytest.mark.parametrize("mode", [0, 1])
def test_select_parity(cuda, ref, mode):
    Hkv, G, R, p0 = 8, 4, 5, 4096
    m, r, q, kn, vn, out, logits, scores, res = _run_verify(ref, Hkv, G, R, [p0], 256, seed=51, score_layout=mode)
    Runner, _, selection_k = _lib()
    l_ref = res[0][1]  # [Hq][R][p0]
    n_sets = 1 if mode == 0 else Hkv
    idx, cnt = _gpu_select(r, 1, mode, n_sets, 2)
    k = selection_k(r.sparse_ratio, p0, r.k_min)
    exact = 0
    for s in range(n_sets):
        heads = range(Hkv * G) if mode == 0 else range(s * G, (s + 1) * G)
        L = l_ref[list(heads)]
        want = ref.select(COLLECT2, L, list(range(1, R + 1)), r.sparse_ratio, r.k_min)
        ref_scores = ref.score_columns(L, list(range(1, R + 1)), [1, R])
        got = idx[0, s, : cnt[0, s]]
        assert cnt[0, s] == k == len(want)
        check_selection(got, ref_scores, k)
        exact += int(np.array_equal(got, want))
    assert exact >= n_sets - 1  # random data: identical sets except at most a rare near-tie


def test_select_exact_ties_lower_index(cuda, ref):
    """Planted exact ties: duplicate key rows give identical scores; the lower index must win."""
    import torch
    Runner, _, selection_k = _lib()
    from paper_2602_07223_b200 import Cache
    Hkv, G, R, p0 = 2, 4, 3, 640
    base = normal_bf16(61, 1, (8, 2 * Hkv, D))
    K = base[np.arange(p0) % 8]  # every key repeats every 8 positions -> massive exact ties
    V = normal_bf16(61, 2, (p0, 2 * Hkv, D))
    cache = Cache(2, Hkv, D, p0 + 64, page_size=128)
    cache.append(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    kv = ref.kv(2, Hkv, D, p0 + 64)
    for t in range(p0):
        kv.append(K[t], V[t])
    r = Runner(cache, Hkv * G, max_rows=R, max_prefix=p0, sparse_ratio=0.1, k_min=16)
    r.set_batch([0], [p0])
    q = normal_bf16(61, 3, (1, Hkv * G, R, D))
    kn, vn = normal_bf16(61, 4, (1, R, Hkv, D)), normal_bf16(61, 5, (1, R, Hkv, D))
    out = torch.zeros((1, Hkv * G, R, D), dtype=torch.float32, device="cuda")
    r.verify(0, to_dev_bf16(q), out, to_dev_bf16(kn), to_dev_bf16(vn), SCALE, score_row_mask=1 | (1 << (R - 1)))
    for t in range(R):
        kk, vv = np.zeros((2 * Hkv, D), np.float32), np.zeros((2 * Hkv, D), np.float32)
        kk[:Hkv], vv[:Hkv] = kn[0, t], vn[0, t]
        kv.append(kk, vv)
    _, l_ref = kv.verify_layer(0, Hkv * G, q[0], p0, R, SCALE, threads=8)
    idx, cnt = _gpu_select(r, 0, 0, 1, 2)
    want = ref.select(COLLECT2, l_ref, list(range(1, R + 1)), 0.1, 16)
    assert cnt[0, 0] == selection_k(0.1, p0, 16) == len(want)
    assert np.array_equal(idx[0, 0, : cnt[0, 0]], want)


@pytest.mark.parametrize("mode", [0, 1])
def test_select_kernels_agree(cuda, ref, mode):
    """The cluster select (8 CTAs, keys in registers, pushed adaptive radix histograms; select_legacy=2)
    and the single-CTA shared-memory radix select (select_legacy=1) give identical index sets and counts
    on the same scores: three sequences with ragged prefixes (one at 40960, past one CTA's register
    span), keys repeating every 16 positions in one of them (exact ties straddling the threshold), both
    score layouts; and the reference's own selection agrees on the tie-heavy sequence."""
    torch = cuda
    Runner, _, selection_k = _lib()
    Hkv, G, R = 2, 4, 3
    p0s = [40960, 9000, 777]
    m = Matched(ref, L=1, Hkv=Hkv, n_tokens=0, seed=66, max_context=max(p0s) + 64, page_size=256,
                n_seqs=3, lens=p0s)
    rep = m.K[1][np.arange(p0s[1]) % 16]  # sequence 1: every key repeats every 16 positions
    m.cache.truncate(0, seq=1)
    m.cache.append(torch.from_numpy(rep).cuda(), torch.from_numpy(m.V[1]).cuda(), seq=1)
    q = normal_bf16(67, 1, (3, Hkv * G, R, D))
    kn, vn = normal_bf16(67, 2, (3, R, Hkv, D)), normal_bf16(67, 3, (3, R, Hkv, D))
    n_sets = 1 if mode == 0 else Hkv
    res = []
    for legacy in (2, 1):  # cluster kernel, single-CTA kernel
        r = Runner(m.cache, Hkv * G, max_rows=R, max_prefix=max(p0s), max_batch=3, sparse_ratio=0.07, k_min=16)
        r.set_dev_knob("select_legacy", legacy)
        r.set_batch([0, 1, 2], p0s)
        out = torch.zeros((3, Hkv * G, R, D), dtype=torch.float32, device="cuda")
        r.verify(0, to_dev_bf16(q), out, to_dev_bf16(kn), to_dev_bf16(vn), SCALE, score_row_mask=1 | (1 << (R - 1)),
                 score_layout=mode)
        for b in range(3):
            m.cache.set_size(p0s[b], seq=b)
        res.append(_gpu_select(r, 0, mode, n_sets, 2))
        r.close()
    (i_new, c_new), (i_old, c_old) = res
    assert np.array_equal(c_new, c_old)
    for b in range(3):
        assert c_new[b, 0] == selection_k(0.07, p0s[b], 16)
        for s_ in range(n_sets):
            assert np.array_equal(i_new[b, s_, :c_new[b, s_]], i_old[b, s_, :c_old[b, s_]]), (b, s_)
    kv = ref.kv(1, Hkv, D, p0s[1] + 64)
    for t in range(p0s[1]):
        kv.append(rep[t], m.V[1][t])
    for t in range(R):
        kv.append(kn[1, t], vn[1, t])
    _, l_ref = kv.verify_layer(0, Hkv * G, q[1], p0s[1], R, SCALE, threads=8)
    for s_ in range(n_sets):
        heads = list(range(Hkv * G)) if mode == 0 else list(range(s_ * G, (s_ + 1) * G))
        want = ref.select(COLLECT2, np.ascontiguousarray(l_ref[heads]), list(range(1, R + 1)), 0.07, 16)
        assert np.array_equal(i_new[1, s_, :c_new[1, s_]], want)


# ----------------------------------------------------------------------------------- draft

# (mode, Hkv, G): G <= 4 runs the packed-plane draft step (P_hi | P_mid share one n8 tile), G = 8 the
# three-mma one; G = 1 and 3 leave padding columns inside the packed tile.  sub > 0 forces the
# two-level merge: `sub` clusters of 4 CTAs per unit, combined through global memory
@pytest.mark.parametrize("mode,Hkv,G,sub", [(0, 8, 4, 0), (1, 8, 4, 0), (0, 2, 1, 0), (0, 4, 3, 0), (1, 2, 8, 0),
                                            (0, 2, 8, 3), (1, 2, 4, 2)])
def test_draft_parity(cuda, ref, mode, Hkv, G, sub):
    torch = cuda
    R, p0 = 5, 4096
    m, r, q, kn, vn, out, logits, scores, res = _run_verify(ref, Hkv, G, R, [p0], 256, seed=71, score_layout=mode)
    if sub:
        r.set_dev_knob("draft_cs", 4)
        r.set_dev_knob("draft_sub", sub)
    n_sets = 1 if mode == 0 else Hkv
    idx, cnt = _gpu_select(r, 1, mode, n_sets, 2)
    sets = [idx[0, s, : cnt[0, s]].astype(np.int64) for s in range(n_sets)]
    kv = m.refs[0]
    kv.truncate(p0)  # draft chain: provisional rows p0.. are re-appended step by step
    m.cache.set_size(p0)
    Hq = Hkv * G
    for step in range(1, R):
        qd = normal_bf16(72, step, (1, Hq, D))
        kd, vd = normal_bf16(73, step, (1, Hkv, D)), normal_bf16(74, step, (1, Hkv, D))
        o = torch.zeros((1, Hq, D), dtype=torch.float32, device="cuda")
        r.draft(1, step, to_dev_bf16(qd), o, to_dev_bf16(kd), to_dev_bf16(vd), mode=mode, scale=SCALE)
        kk, vv = np.zeros((2 * Hkv, D), np.float32), np.zeros((2 * Hkv, D), np.float32)
        kk[Hkv:], vv[Hkv:] = kd[0], vd[0]
        kv.append(kk, vv)
        o_ref = kv.draft_layer(1, Hq, qd[0], sets, p0, step, SCALE, threads=8)
        got = o.cpu().numpy()[0]
        assert rel_err_rows(got, o_ref) < 2e-4, (step, rel_err_rows(got, o_ref))
        assert rel_err_elem(got, o_ref) < 2e-3


# ----------------------------------------------------------------------------------- iteration

ITERATION_CASES = [(COLLECT2, 0, True, 0, 0), (ALL_DRAFT, 1, False, 0, 0), (LAST_ACCEPTED, 0, True, 2, 0),
                   (COLLECT2, 0, True, 4, 0),
                   # the batched selection schedule (dev knob select_batched: every layer's top-k in one
                   # grid-z launch after the verify chain, one dependency edge into the draft chain)
                   (COLLECT2, 0, True, 1, 1), (ALL_DRAFT, 1, False, 3, 1), (LAST_ACCEPTED, 0, True, 2, 1)]


@pytest.mark.parametrize("strategy,mode,use_graph,accepted,batched", ITERATION_CASES)
def test_iteration_parity(cuda, ref, strategy, mode, use_graph, accepted, batched):
    """One full speculation iteration (verify -> select -> gamma drafts, all layers) through
    sa_iteration_run vs the reference composition (SURVEY.md §8d unit of work).  The draft phase is the
    next draft chain after accepting a = `accepted` drafts: its rows go to p0+a+1.. and its tail is
    [p0, p0+a+1+j); the commit afterwards keeps the verify's rows p0..p0+a."""
    torch = cuda
    Runner, _, selection_k = _lib()
    L, Hkv, G, gamma, p0 = 3, 2, 4, 4, 1200
    R, Hq = gamma + 1, Hkv * G
    m = Matched(ref, L=L, Hkv=Hkv, n_tokens=p0, seed=81, max_context=p0 + 64, page_size=128)
    r = Runner(m.cache, Hq, max_rows=R, max_prefix=p0, sparse_ratio=0.07, k_min=16)
    if batched:
        r.set_dev_knob("select_batched", 1)
    r.set_batch([0], [p0])
    qv = normal_bf16(82, 1, (L, 1, Hq, R, D))
    kvn, vvn = normal_bf16(82, 2, (L, 1, R, Hkv, D)), normal_bf16(82, 3, (L, 1, R, Hkv, D))
    qd = normal_bf16(82, 4, (gamma, L, 1, Hq, D))
    kdn, vdn = normal_bf16(82, 5, (gamma, L, 1, Hkv, D)), normal_bf16(82, 6, (gamma, L, 1, Hkv, D))
    out_v = torch.zeros((L, 1, Hq, R, D), dtype=torch.float32, device="cuda")
    out_d = torch.zeros((gamma, L, 1, Hq, D), dtype=torch.float32, device="cuda")
    dev = [to_dev_bf16(x) for x in (qv, kvn, vvn, qd, kdn, vdn)]
    args = r.iteration_args(gamma, *dev, out_v, out_d, strategy=strategy, mode=mode, scale=SCALE,
                            use_graph=use_graph, accepted=accepted)
    assert r.iteration_kernel_count(args) == L * (2 + gamma)
    for _ in range(2):  # second launch replays the graph
        r.iteration(args)
    torch.cuda.synchronize()
    ov, od = out_v.cpu().numpy(), out_d.cpu().numpy()
    kv = m.refs[0]
    for t in range(R):
        kv.append(kvn[:, 0, t].reshape(L * Hkv, D), vvn[:, 0, t].reshape(L * Hkv, D))
    n_sets = 1 if mode == 0 else Hkv
    rows = {COLLECT2: [1, R], ALL_DRAFT: list(range(1, R + 1)), LAST_ACCEPTED: [accepted + 1]}[strategy]
    k = selection_k(0.07, p0, 16)
    sets_by_layer = []
    for layer in range(L):
        o_ref, l_ref = kv.verify_layer(layer, Hq, qv[layer, 0], p0, R, SCALE, threads=8)
        assert rel_err_rows(ov[layer, 0], o_ref) < 2e-4
        idx, cnt = r.selection(layer, n_sets)
        sets = []
        for s in range(n_sets):
            heads = list(range(Hq)) if mode == 0 else list(range(s * G, (s + 1) * G))
            sc = ref.score_columns(l_ref[heads], list(range(1, R + 1)), rows)
            got = idx[0, s, : cnt[0, s]]
            check_selection(got, sc, k)
            if strategy == LAST_ACCEPTED and mode == 0:  # the reference entry point itself (selection.cpp:198-207)
                want = ref.select(LAST_ACCEPTED, l_ref, list(range(1, R + 1)), 0.07, 16, accepted=accepted)
                assert len(want) == len(got) and len(set(want.tolist()) ^ set(got.tolist())) <= 2
            sets.append(got.astype(np.int64))
        sets_by_layer.append(sets)
    # the next draft chain: the reference keeps [y, x1..xa] (p0..p0+a), then appends the draft rows; the
    # draft query of step j attends to T and the tail [p0, p0+a+1+j)
    a = accepted
    kv.truncate(p0 + a + 1)
    for j in range(1, gamma + 1):
        kv.append(kdn[j - 1, :, 0].reshape(L * Hkv, D), vdn[j - 1, :, 0].reshape(L * Hkv, D))
        for layer in range(L):
            o_ref = kv.draft_layer(layer, Hq, qd[j - 1, layer, 0], sets_by_layer[layer], p0, a + 1 + j, SCALE,
                                   threads=8)
            assert rel_err_rows(od[j - 1, layer, 0], o_ref) < 2e-4, (j, layer)
            assert rel_err_elem(od[j - 1, layer, 0], o_ref) < 2e-3, (j, layer)
    # commit a: the store keeps the verify's rows p0..p0+a, not the draft chain's provisional rows
    m.cache.commit_accepted(p0, a)
    assert m.cache.size() == p0 + a + 1
    for layer in range(L):
        for h in range(Hkv):
            K, V = m.cache.read(layer, h, p0, a + 1)
            assert np.array_equal(K.cpu().numpy(), kvn[layer, 0, : a + 1, h]), (layer, h)
            assert np.array_equal(V.cpu().numpy(), vvn[layer, 0, : a + 1, h]), (layer, h)


# ----------------------------------------------------------------------------------- sharding

def test_head_sharded_layer_scores_sum_exactly(cuda):
    """KV-head sharding with real kernels on one GPU: two half-head caches (the two
    ranks' shards) produce per-layer fixed-point sums whose integer sum is bit-identical to the
    full cache's, and selecting on the exchanged sums gives the full cache's selection exactly."""
    torch = cuda
    from paper_2602_07223_b200 import Cache, Runner
    L, Hkv, G, R, p0 = 1, 4, 4, 5, 2500
    Hq = Hkv * G
    K = normal_bf16(95, 1, (p0, L * Hkv, D))
    V = normal_bf16(95, 2, (p0, L * Hkv, D))
    q = normal_bf16(95, 3, (1, Hq, R, D))
    kn, vn = normal_bf16(95, 4, (1, R, Hkv, D)), normal_bf16(95, 5, (1, R, Hkv, D))

    def run(heads):
        c = Cache(L, len(heads), D, p0 + 64, page_size=128)
        c.append(torch.from_numpy(np.ascontiguousarray(K[:, heads])).cuda(),
                 torch.from_numpy(np.ascontiguousarray(V[:, heads])).cuda())
        r = Runner(c, len(heads) * G, max_rows=R, max_prefix=p0)
        r.set_batch([0], [p0])
        qh = np.ascontiguousarray(q[:, heads[0] * G:(heads[-1] + 1) * G])
        out = torch.zeros((1, len(heads) * G, R, D), dtype=torch.float32, device="cuda")
        r.verify(0, to_dev_bf16(qh), out, to_dev_bf16(np.ascontiguousarray(kn[:, :, heads])),
                 to_dev_bf16(np.ascontiguousarray(vn[:, :, heads])), SCALE)
        torch.cuda.synchronize()
        return c, r

    full = run([0, 1, 2, 3])
    a, b = run([0, 1]), run([2, 3])
    fx_full = full[1].layer_scores(0)
    fx_a, fx_b = a[1].layer_scores(0), b[1].layer_scores(0)
    assert np.array_equal(fx_full, fx_a + fx_b)
    # the exchange (what shard.exchange_layer_scores' all-reduce does), in place on shard a's buffer
    ta = a[1].layer_scores_tensor(0)
    ta += torch.from_numpy(fx_b).cuda()
    torch.cuda.synchronize()
    full[1].select(0)
    a[1].select(0)
    i_full, c_full = full[1].selection(0, 1)
    i_a, c_a = a[1].selection(0, 1)
    assert c_full[0, 0] == c_a[0, 0] and np.array_equal(i_full[0, 0, :c_full[0, 0]], i_a[0, 0, :c_a[0, 0]])


def test_iteration_with_score_exchange(cuda):
    """§8e exchange wired into the iteration graph: a KV-head group communicator (one rank here, a
    real NCCL communicator: the all-reduce runs inside the captured graph between every layer's
    verify and select) leaves the selections bit-identical to a run without it."""
    torch = cuda
    from paper_2602_07223_b200 import Cache, Comm, Runner
    L, Hkv, G, gamma, p0 = 2, 2, 4, 4, 1500
    R, Hq = gamma + 1, Hkv * G
    K = normal_bf16(97, 1, (p0, L * Hkv, D))
    V = normal_bf16(97, 2, (p0, L * Hkv, D))
    ins = [to_dev_bf16(normal_bf16(97, 3 + i, s)) for i, s in enumerate(
        [(L, 1, Hq, R, D), (L, 1, R, Hkv, D), (L, 1, R, Hkv, D), (gamma, L, 1, Hq, D), (gamma, L, 1, Hkv, D),
         (gamma, L, 1, Hkv, D)])]

    def run(comm):
        c = Cache(L, Hkv, D, p0 + 64, page_size=128)
        c.append(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
        r = Runner(c, Hq, max_rows=R, max_prefix=p0)
        r.set_batch([0], [p0])
        if comm is not None:
            r.set_comm(comm)
        ov = torch.zeros((L, 1, Hq, R, D), dtype=torch.float32, device="cuda")
        od = torch.zeros((gamma, L, 1, Hq, D), dtype=torch.float32, device="cuda")
        a = r.iteration_args(gamma, *ins, ov, od, scale=SCALE, use_graph=True)
        for _ in range(2):
            r.iteration(a)
        torch.cuda.synchronize()
        return [r.selection(l, 1) for l in range(L)], ov.cpu().numpy(), od.cpu().numpy()

    comm = Comm(Comm.unique_id(), 1, 0)
    base, with_comm = run(None), run(comm)
    for (i0, c0), (i1, c1) in zip(base[0], with_comm[0]):
        assert np.array_equal(c0, c1) and np.array_equal(i0, i1)
    assert np.array_equal(base[1], with_comm[1]) and np.array_equal(base[2], with_comm[2])


@pytest.mark.parametrize("mode", [0, 1])
def test_collect2_weights_selection(cuda, ref, mode):
    """Collect2Weights (score_columns_weights, selection.cpp:110-135): softmax-weight scores from the
    verify kernel's raw logits of rows {1, gamma+1}, then top-k — vs the reference's select."""
    torch = cuda
    from oracle.pyoracle import COLLECT2_WEIGHTS
    Hkv, G, R, p0 = 4, 4, 5, 3000
    m, r, q, kn, vn, out, logits, scores, res = _run_verify(ref, Hkv, G, R, [p0], 256, seed=53, score_layout=mode)
    l_ref = res[0][1]
    _, _, selection_k = _lib()
    lg = torch.from_numpy(np.ascontiguousarray(logits[:, :, [0, R - 1], :])).cuda()
    r.score_weights(1, lg, 2, mode=mode)
    n_sets = 1 if mode == 0 else Hkv
    r.select(1, mode=mode, rows_in_score=2)
    idx, cnt = r.selection(1, n_sets)
    k = selection_k(r.sparse_ratio, p0, r.k_min)
    exact = 0
    for s in range(n_sets):
        heads = list(range(Hkv * G)) if mode == 0 else list(range(s * G, (s + 1) * G))
        L = l_ref[heads]
        want = ref.select(COLLECT2_WEIGHTS, L, list(range(1, R + 1)), r.sparse_ratio, r.k_min, head_dim=D)
        sc = ref.score_columns(L, list(range(1, R + 1)), [1, R], weights=True, head_dim=D)
        got = idx[0, s, : cnt[0, s]]
        assert cnt[0, s] == k == len(want)
        check_selection(got, sc, k, relative=True)
        exact += int(np.array_equal(got, want))
    assert exact >= n_sets - 1


def test_iteration_collect2_weights(cuda, ref):
    """The weights metric inside the iteration graph (verify -> raw logits -> weights -> select)."""
    torch = cuda
    from oracle.pyoracle import COLLECT2_WEIGHTS
    Runner, _, selection_k = _lib()
    L, Hkv, G, gamma, p0 = 2, 2, 4, 4, 1100
    R, Hq = gamma + 1, Hkv * G
    m = Matched(ref, L=L, Hkv=Hkv, n_tokens=p0, seed=87, max_context=p0 + 64, page_size=128)
    r = Runner(m.cache, Hq, max_rows=R, max_prefix=p0, sparse_ratio=0.07, k_min=16)
    r.set_batch([0], [p0])
    qv = normal_bf16(88, 1, (L, 1, Hq, R, D))
    kvn, vvn = normal_bf16(88, 2, (L, 1, R, Hkv, D)), normal_bf16(88, 3, (L, 1, R, Hkv, D))
    qd = normal_bf16(88, 4, (gamma, L, 1, Hq, D))
    kdn, vdn = normal_bf16(88, 5, (gamma, L, 1, Hkv, D)), normal_bf16(88, 6, (gamma, L, 1, Hkv, D))
    out_v = torch.zeros((L, 1, Hq, R, D), dtype=torch.float32, device="cuda")
    out_d = torch.zeros((gamma, L, 1, Hq, D), dtype=torch.float32, device="cuda")
    dev = [to_dev_bf16(x) for x in (qv, kvn, vvn, qd, kdn, vdn)]
    args = r.iteration_args(gamma, *dev, out_v, out_d, strategy=COLLECT2_WEIGHTS, scale=SCALE, use_graph=True)
    assert r.iteration_kernel_count(args) == L * (4 + gamma)
    for _ in range(2):
        r.iteration(args)
    torch.cuda.synchronize()
    kv = m.refs[0]
    for t in range(R):
        kv.append(kvn[:, 0, t].reshape(L * Hkv, D), vvn[:, 0, t].reshape(L * Hkv, D))
    k = selection_k(0.07, p0, 16)
    for layer in range(L):
        o_ref, l_ref = kv.verify_layer(layer, Hq, qv[layer, 0], p0, R, SCALE, threads=8)
        assert rel_err_rows(out_v.cpu().numpy()[layer, 0], o_ref) < 2e-4
        idx, cnt = r.selection(layer, 1)
        sc = ref.score_columns(l_ref, list(range(1, R + 1)), [1, R], weights=True, head_dim=D)
        check_selection(idx[0, 0, : cnt[0, 0]], sc, k, relative=True)


# knobs: automatic (the streaming mode here), or forced CTAs per unit in the two-CTA-per-SM mode with
# several rounds: 4 CTAs -> <= 4 rounds of 96 rows, all resolved before the wait (slots 0 and 1 gathered
# early); 2 CTAs -> up to 8 rounds (resolved per round after the wait), double-buffered 96-row slots
@pytest.mark.parametrize("knobs", [{}, {"draft_cs": 4}, {"draft_cs": 2}])
def test_draft_streaming_mode(cuda, ref, knobs):
    """Draft launches whose chunks span several resident rounds (large k x many sequences: the
    streaming mode, one CTA per SM with double-buffered rounds, or forced multi-round clusters at two
    CTAs per SM) vs the reference gather + attend."""
    torch = cuda
    Runner, _, selection_k = _lib()
    Hkv, G, R, B = 8, 4, 3, 6
    p0s = [2600, 3000, 1900, 2800, 3000, 2200]
    Hq = Hkv * G
    m = Matched(ref, L=2, Hkv=Hkv, n_tokens=0, seed=61, max_context=max(p0s) + 64, page_size=128, n_seqs=B,
                lens=p0s)
    r = Runner(m.cache, Hq, max_rows=R, max_prefix=max(p0s), max_batch=B, sparse_ratio=0.5, k_min=16)
    for kname, kval in knobs.items():
        r.set_dev_knob(kname, kval)
    r.set_batch(list(range(B)), p0s)
    q = normal_bf16(62, 1, (B, Hq, R, D))
    kn, vn = normal_bf16(62, 2, (B, R, Hkv, D)), normal_bf16(62, 3, (B, R, Hkv, D))
    out = torch.zeros((B, Hq, R, D), dtype=torch.float32, device="cuda")
    r.verify(1, to_dev_bf16(q), out, to_dev_bf16(kn), to_dev_bf16(vn), SCALE)
    r.select(1)
    idx, cnt = r.selection(1, 1)
    for b in range(B):
        assert cnt[b, 0] == selection_k(0.5, p0s[b], 16)
        m.cache.set_size(p0s[b], seq=b)
    for step in range(1, R):  # step 2 also gathers the tail row step 1 appended (old-tail path)
        qd = normal_bf16(63, 10 * step + 1, (B, Hq, D))
        kd, vd = normal_bf16(63, 10 * step + 2, (B, Hkv, D)), normal_bf16(63, 10 * step + 3, (B, Hkv, D))
        od = torch.zeros((B, Hq, D), dtype=torch.float32, device="cuda")
        r.draft(1, step, to_dev_bf16(qd), od, to_dev_bf16(kd), to_dev_bf16(vd), scale=SCALE)
        got = od.cpu().numpy()
        for b in range(B):
            kv = m.refs[b]
            kk, vv = np.zeros((2 * Hkv, D), np.float32), np.zeros((2 * Hkv, D), np.float32)
            kk[Hkv:], vv[Hkv:] = kd[b], vd[b]
            kv.append(kk, vv)
            sets = [idx[b, 0, : cnt[b, 0]].astype(np.int64)]
            o_ref = kv.draft_layer(1, Hq, qd[b], sets, p0s[b], step, SCALE, threads=8)
            assert rel_err_rows(got[b], o_ref) < 2e-4, (step, b, rel_err_rows(got[b], o_ref))
            assert rel_err_elem(got[b], o_ref) < 2e-3


def test_quest_and_window_selectors(cuda, ref):
    """Baseline selectors on the GPU vs the reference's own select_quest / select_window
    (selection.cpp:209-274) over page summaries maintained like KvStore's (kv_store.cpp:90-139),
    including a lazy refresh after appends; the draft kernel consumes the Quest set."""
    torch = cuda
    from oracle.pyoracle import quest_bounds, ref_select_window
    Runner, _, selection_k = _lib()
    L, Hkv, G, p0, page = 2, 4, 4, 2000, 8
    Hq = Hkv * G
    m = Matched(ref, L=L, Hkv=Hkv, n_tokens=p0, seed=111, max_context=p0 + 200, page_size=128)
    kv = m.refs[0]
    kv.enable_page_summaries(page)
    m.cache.enable_page_summaries(page)
    r = Runner(m.cache, Hq, max_rows=5, max_prefix=p0 + 100, sparse_ratio=0.1, k_min=16)

    def check(prefix, layer, seed):
        r.set_batch([0], [prefix])
        q = normal_bf16(seed, layer, (1, Hq, D))
        r.select_quest(layer, to_dev_bf16(q))
        idx, cnt = r.selection(layer, 1)
        got = idx[0, 0, : cnt[0, 0]]
        want = kv.select_quest(q[0], layer, prefix, 0.1, 16)
        assert cnt[0, 0] == selection_k(0.1, prefix, 16) == len(want)
        if not np.array_equal(got, want):  # only near-tied page bounds may differ (fp32 sum order)
            mins = np.stack([kv.page_minmax(layer, g)[0] for g in range(Hkv)])
            maxs = np.stack([kv.page_minmax(layer, g)[1] for g in range(Hkv)])
            n_pages = (prefix + page - 1) // page
            b = quest_bounds(mins[:, :n_pages], maxs[:, :n_pages], q[0], G)
            diff = set(got.tolist()) ^ set(want.tolist())
            pages = {i // page for i in diff}
            b_last = min(b[i // page] for i in want)
            assert all(abs(b[pp] - b_last) <= 1e-4 * max(abs(b_last), 1.0) for pp in pages), sorted(pages)
        return got, q

    check(p0, 1, 5)
    check(1500, 0, 6)
    # appends (the summaries' tail pages go stale and are rebuilt lazily on the next selection)
    extra = normal_bf16(112, 1, (60, L * Hkv, D))
    m.cache.append(torch.from_numpy(extra).cuda(), torch.from_numpy(extra).cuda())
    for t in range(60):
        kv.append(extra[t], extra[t])
    got, q = check(p0 + 60, 1, 7)
    # the draft kernel over the Quest set (gather(T) ++ tail, then attend)
    qd = normal_bf16(113, 1, (1, Hq, D))
    kd, vd = normal_bf16(113, 2, (1, Hkv, D)), normal_bf16(113, 3, (1, Hkv, D))
    od = torch.zeros((1, Hq, D), dtype=torch.float32, device="cuda")
    r.draft(1, 1, to_dev_bf16(qd), od, to_dev_bf16(kd), to_dev_bf16(vd), scale=SCALE)
    kk, vv = np.zeros((L * Hkv, D), np.float32), np.zeros((L * Hkv, D), np.float32)
    kk[Hkv:], vv[Hkv:] = kd[0], vd[0]
    kv.append(kk, vv)
    o_ref = kv.draft_layer(1, Hq, qd[0], [got.astype(np.int64)], p0 + 60, 1, SCALE, threads=8)
    assert rel_err_rows(od.cpu().numpy()[0], o_ref) < 2e-4
    # window selector
    r.set_batch([0], [p0])
    r.select_window(1, sink=4, window=150)
    idx, cnt = r.selection(1, 1)
    assert np.array_equal(idx[0, 0, : cnt[0, 0]], ref_select_window(ref, p0, 4, 150))


@pytest.mark.parametrize("strategy", ["quest", "window"])
def test_iteration_baseline_strategies(cuda, ref, strategy):
    """The iteration with the paper's baselines: QuestLike re-selects before every draft launch from
    that step's query, Window once per iteration (sink 4 + window k - 4)."""
    torch = cuda
    from oracle.pyoracle import ref_select_window
    from paper_2602_07223_b200 import QUEST_LIKE, WINDOW
    Runner, _, selection_k = _lib()
    L, Hkv, G, gamma, p0 = 2, 2, 4, 3, 1600
    R, Hq = gamma + 1, Hkv * G
    m = Matched(ref, L=L, Hkv=Hkv, n_tokens=p0, seed=121, max_context=p0 + 64, page_size=128)
    kv = m.refs[0]
    if strategy == "quest":
        m.cache.enable_page_summaries(8)
        kv.enable_page_summaries(8)
    r = Runner(m.cache, Hq, max_rows=R, max_prefix=p0, sparse_ratio=0.07, k_min=16)
    r.set_batch([0], [p0])
    qv = normal_bf16(122, 1, (L, 1, Hq, R, D))
    kvn, vvn = normal_bf16(122, 2, (L, 1, R, Hkv, D)), normal_bf16(122, 3, (L, 1, R, Hkv, D))
    qd = normal_bf16(122, 4, (gamma, L, 1, Hq, D))
    kdn, vdn = normal_bf16(122, 5, (gamma, L, 1, Hkv, D)), normal_bf16(122, 6, (gamma, L, 1, Hkv, D))
    out_v = torch.zeros((L, 1, Hq, R, D), dtype=torch.float32, device="cuda")
    out_d = torch.zeros((gamma, L, 1, Hq, D), dtype=torch.float32, device="cuda")
    dev = [to_dev_bf16(x) for x in (qv, kvn, vvn, qd, kdn, vdn)]
    st = QUEST_LIKE if strategy == "quest" else WINDOW
    args = r.iteration_args(gamma, *dev, out_v, out_d, strategy=st, scale=SCALE, use_graph=True)
    for _ in range(2):
        r.iteration(args)
    torch.cuda.synchronize()
    k = selection_k(0.07, p0, 16)
    for t in range(R):
        kv.append(kvn[:, 0, t].reshape(L * Hkv, D), vvn[:, 0, t].reshape(L * Hkv, D))
    for layer in range(L):  # verify outputs are strategy-independent
        o_ref, _ = kv.verify_layer(layer, Hq, qv[layer, 0], p0, R, SCALE, want_logits=False, threads=8)
        assert rel_err_rows(out_v.cpu().numpy()[layer, 0], o_ref) < 2e-4
    a = 0  # sa_iteration_args.accepted: the next draft chain starts at p0 + a + 1 (after y)
    kv.truncate(p0 + a + 1)
    od = out_d.cpu().numpy()
    for j in range(1, gamma + 1):
        kv.append(kdn[j - 1, :, 0].reshape(L * Hkv, D), vdn[j - 1, :, 0].reshape(L * Hkv, D))
        for layer in range(L):
            if strategy == "window":
                T = ref_select_window(ref, p0, 4, k - 4)
            else:  # the set the reference picks from this step's query (summaries over the store)
                T = kv.select_quest(qd[j - 1, layer, 0], layer, p0, 0.07, 16)
            o_ref = kv.draft_layer(layer, Hq, qd[j - 1, layer, 0], [T], p0, a + 1 + j, SCALE, threads=8)
            assert rel_err_rows(od[j - 1, layer, 0], o_ref) < 2e-4, (j, layer)
            assert rel_err_elem(od[j - 1, layer, 0], o_ref) < 2e-3, (j, layer)
    idx, cnt = r.selection(L - 1, 1)
    assert cnt[0, 0] == k


# ----------------------------------------------------------------------- speculation glue (§8f)

def _spec_case(rng, B, g, V, temp=1.0):
    z = rng.standard_normal((B, 1, V)) * 2.0
    p = np.exp(z + temp * rng.standard_normal((B, g + 1, V)))
    q = np.exp(z + temp * rng.standard_normal((B, g, V)))
    p = (p / p.sum(-1, keepdims=True)).astype(np.float32)
    q = (q / q.sum(-1, keepdims=True)).astype(np.float32)
    cq = np.cumsum(q.astype(np.float64), -1)
    draft = np.minimum((cq < rng.random((B, g, 1)) * cq[..., -1:]).sum(-1), V - 1).astype(np.int32)
    u = rng.random((B, g + 1)).astype(np.float32)
    return p, q, draft, u


@pytest.mark.parametrize("B,g,V", [(256, 4, 1000), (8, 3, 50000), (64, 1, 7)])
def test_accept_parity(cuda, B, g, V):
    torch = cuda
    from oracle.speculation import accept as ref_accept
    from paper_2602_07223_b200 import accept
    rng = np.random.default_rng(B + V)
    p, q, draft, u = _spec_case(rng, B, g, V)
    acc, em = accept(*(torch.from_numpy(x).cuda() for x in (p, draft)), q=torch.from_numpy(q).cuda(),
                     u=torch.from_numpy(u).cuda())
    acc, em = acc.cpu().numpy(), em.cpu().numpy()
    seen = set()
    for b in range(B):
        a, e = ref_accept(p[b], draft[b], q=q[b], u=u[b])
        assert acc[b] == a and list(em[b, :a + 1]) == e, b
        assert np.all(em[b, a + 1:] == -1)
        seen.add(a)
    if B >= 64:
        assert len(seen) >= 2  # both accept and reject paths exercised


def test_accept_greedy_ties(cuda):
    torch = cuda
    from oracle.speculation import accept as ref_accept
    from paper_2602_07223_b200 import accept
    rng = np.random.default_rng(4)
    B, g, V = 64, 4, 5000
    p = rng.integers(0, 4, size=(B, g + 1, V)).astype(np.float32)  # many exact ties at the max
    draft = np.argmax(p[:, :g], -1).astype(np.int32)
    flip = rng.random((B, g)) < 0.3
    draft[flip] = rng.integers(0, V, size=flip.sum())
    acc, em = accept(torch.from_numpy(p).cuda(), torch.from_numpy(draft).cuda(), greedy=True)
    acc, em = acc.cpu().numpy(), em.cpu().numpy()
    for b in range(B):
        a, e = ref_accept(p[b], draft[b], greedy=True)
        assert acc[b] == a and list(em[b, :a + 1]) == e


def test_accept_emission_distribution(cuda):
    # empirical single-step emission distribution over 100000 seeded runs matches p, TV < 0.01
    torch = cuda
    from paper_2602_07223_b200 import accept
    rng = np.random.default_rng(12)
    B, V = 100000, 8
    p1 = rng.dirichlet(np.ones(V)).astype(np.float32)
    q1 = rng.dirichlet(np.ones(V)).astype(np.float32)
    p = np.broadcast_to(p1, (B, 2, V)).copy()
    q = np.broadcast_to(q1, (B, 1, V)).copy()
    cq = np.cumsum(q1.astype(np.float64))
    draft = np.minimum(np.searchsorted(cq / cq[-1], rng.random((B, 1)), side="right"), V - 1).astype(np.int32)
    u = rng.random((B, 2)).astype(np.float32)
    acc, em = accept(*(torch.from_numpy(x).cuda() for x in (p, draft)), q=torch.from_numpy(q).cuda(),
                     u=torch.from_numpy(u).cuda())
    first = em[:, 0].cpu().numpy()
    freq = np.bincount(first, minlength=V) / B
    assert 0.5 * np.abs(freq - p1).sum() < 0.01
    rate = acc.float().mean().item()
    assert abs(rate - np.minimum(p1, q1).sum()) < 0.01  # E[accept] = sum_x min(p, q)


def test_commit_accepted(cuda, ref):
    torch = cuda
    from paper_2602_07223_b200 import Cache, SpecAttnError
    c = Cache(1, 1, max_context=256, page_size=128)
    try:
        k = torch.randn(10, 1, 128, device="cuda").to(torch.bfloat16)
        c.append(k, k.clone())
        c.set_committed(5)
        c.commit_accepted(5, 2)  # verify rows 5..9 = [y, x1..x4]; a = 2 keeps 5,6,7
        assert c.size() == 8 and c.committed() == 8
        with pytest.raises(SpecAttnError):
            c.commit_accepted(200, 100)  # beyond the reserved rows
    finally:
        c.close()


# ----------------------------------------------------------------- model-side producer (§8f rank 4)

def _bf16_round(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).float().numpy()


@pytest.mark.parametrize("D,Hq,Hkv,B,rows,style", [
    (256, 8, 2, 1, 5, 0),       # reference toy config (config.hpp:52-54)
    (4096, 32, 8, 1, 5, 0),     # Llama-3.1-8B shape, verify rows
    (4096, 32, 8, 4, 1, 1),     # draft rows, interleaved RoPE
    (1024, 8, 2, 16, 5, 0),     # 80 tokens
    (512, 4, 4, 32, 4, 1),      # 128 tokens (the per-call maximum)
])
def test_qkv_projection_parity(cuda, D, Hq, Hkv, B, rows, style):
    torch = cuda
    from oracle.model import qkv_project
    from paper_2602_07223_b200 import QkvProjection
    rng = np.random.default_rng(D + B * rows + style)
    L, n_out = 2, (Hq + 2 * Hkv) * 128
    w = _bf16_round(rng.standard_normal((L, n_out, D)) / np.sqrt(D))  # N(0, 1/fan_in), weights.hpp:39
    gain = (1.0 + 0.1 * rng.standard_normal((L, D))).astype(np.float32)
    x = rng.standard_normal((B, rows, D)).astype(np.float32) * 3.0
    pos = rng.integers(0, 131072 - rows, size=B).astype(np.int32)
    proj = QkvProjection(torch.from_numpy(w).to(torch.bfloat16).cuda(), torch.from_numpy(gain).cuda(), Hq, Hkv,
                         rope_style=style)
    for layer in range(L):
        q, k, v = proj.project(layer, torch.from_numpy(x).cuda(), torch.from_numpy(pos).cuda())
        torch.cuda.synchronize()
        rq, rk, rv = qkv_project(x, w[layer], gain[layer], Hq, Hkv, pos, style=style)
        for got, ref in ((q, rq), (k, rk), (v, rv)):
            got = got.float().cpu().numpy()
            scale = np.sqrt(np.mean(ref * ref, axis=-1, keepdims=True))
            err = np.abs(got - ref)
            assert np.all(err <= 2.0 ** -8 * np.abs(ref) + 1e-5 * scale), err.max()
            # the fp32-accurate product rounds like the exact value except within ~1e-5 of a tie
            assert np.mean(got == _bf16_round(ref)) > 0.995
    proj.close()


def test_qkv_projection_deterministic_and_errors(cuda):
    torch = cuda
    from paper_2602_07223_b200 import QkvProjection, SpecAttnError
    rng = np.random.default_rng(8)
    w = torch.from_numpy(_bf16_round(rng.standard_normal((1, 12 * 128, 512)) / 23)).to(torch.bfloat16).cuda()
    proj = QkvProjection(w, torch.ones(1, 512, device="cuda"), 8, 2)
    x = torch.randn(2, 5, 512, device="cuda")
    pos = torch.tensor([100, 7], dtype=torch.int32, device="cuda")
    a = [t.clone() for t in proj.project(0, x, pos)]
    b = proj.project(0, x, pos)
    assert all(torch.equal(u, v) for u, v in zip(a, b))
    with pytest.raises(SpecAttnError):
        proj.project(1, x, pos)  # layer out of range
    with pytest.raises(SpecAttnError):
        proj.project(0, torch.randn(2, 65, 512, device="cuda"), pos)  # > 128 tokens
    proj.close()


def test_producer_feeds_verify_and_commit(cuda, ref):
    """The §8f producer's q / k_new / v_new drive the verify kernel directly (layouts end to end), the
    acceptance kernel decides, and commit_accepted leaves the cache at p0 + a + 1."""
    torch = cuda
    from oracle.model import qkv_project
    from oracle.speculation import accept as ref_accept
    from paper_2602_07223_b200 import QkvProjection, accept
    Runner, _, _ = _lib()
    Hkv, G, R, p0, Dm = 2, 4, 5, 300, 256
    Hq = Hkv * G
    m = Matched(ref, L=2, Hkv=Hkv, n_tokens=p0, seed=41, max_context=p0 + R + 64, page_size=128)
    rng = np.random.default_rng(41)
    w = rng.standard_normal((2, (Hq + 2 * Hkv) * 128, Dm)).astype(np.float32) / 16
    w = torch.from_numpy(w).to(torch.bfloat16)
    gain = (1 + 0.1 * rng.standard_normal((2, Dm))).astype(np.float32)
    proj = QkvProjection(w.cuda(), torch.from_numpy(gain).cuda(), Hq, Hkv)
    x = rng.standard_normal((1, R, Dm)).astype(np.float32)
    q, kn, vn = proj.project(1, torch.from_numpy(x).cuda(), torch.tensor([p0], dtype=torch.int32, device="cuda"))
    r = Runner(m.cache, Hq, max_rows=R, max_prefix=p0)
    r.set_batch([0], [p0])
    out = torch.zeros((1, Hq, R, D), dtype=torch.float32, device="cuda")
    r.verify(1, q, out, kn, vn, SCALE, score_row_mask=1 | (1 << (R - 1)))
    torch.cuda.synchronize()
    # producer outputs vs the float64 restatement (half a bf16 ulp + fp32 slack)
    rq, rk, _ = qkv_project(x, w[1].float().numpy(), gain[1], Hq, Hkv, [p0])
    assert np.all(np.abs(q.float().cpu().numpy() - rq) <= 2.0 ** -8 * np.abs(rq) + 1e-4)
    assert np.all(np.abs(kn.float().cpu().numpy() - rk) <= 2.0 ** -8 * np.abs(rk) + 1e-4)
    # verify over the producer's exact bf16 values vs the reference TUs
    qh, kh, vh = (t.float().cpu().numpy() for t in (q, kn, vn))
    kv = m.refs[0]
    for t in range(R):
        kk = np.zeros((2 * Hkv, D), np.float32)
        vv = np.zeros((2 * Hkv, D), np.float32)
        kk[Hkv:], vv[Hkv:] = kh[0, t], vh[0, t]
        kv.append(kk, vv)
    o_ref, _ = kv.verify_layer(1, Hq, qh[0], p0, R, SCALE, threads=8)
    assert rel_err_rows(out.cpu().numpy()[0], o_ref) < 2e-4
    # acceptance on the device, then commit: the store keeps [y, x_1..x_a] and drops the rest
    V = 64
    pp = rng.dirichlet(np.ones(V), size=(1, R)).astype(np.float32)
    qq = rng.dirichlet(np.ones(V), size=(1, R - 1)).astype(np.float32)
    xx = rng.integers(0, V, size=(1, R - 1)).astype(np.int32)
    uu = rng.random((1, R)).astype(np.float32)
    acc, em = accept(*(torch.from_numpy(a_).cuda() for a_ in (pp, xx)), q=torch.from_numpy(qq).cuda(),
                     u=torch.from_numpy(uu).cuda())
    a_ref, e_ref = ref_accept(pp[0], xx[0], q=qq[0], u=uu[0])
    a = int(acc.item())
    assert a == a_ref and list(em.cpu().numpy()[0, :a + 1]) == e_ref
    m.cache.commit_accepted(p0, a)
    assert m.cache.size() == p0 + a + 1 and m.cache.committed() == p0 + a + 1
    proj.close()


def test_quest_all_bounds_tied(cuda, ref):
    """Every page bound equal (constant keys): the candidate set is every page and the reference's
    tie rule (lower page first) decides alone; a partial last page included."""
    torch = cuda
    Runner, _, selection_k = _lib()
    from paper_2602_07223_b200 import Cache
    L, Hkv, G, p0, page = 2, 2, 4, 1003, 8
    Hq = Hkv * G
    K = np.full((p0, L * Hkv, D), 0.5, np.float32)
    V = normal_bf16(5, 2, (p0, L * Hkv, D))
    kv = ref.kv(L, Hkv, D, p0 + 64)
    for t in range(p0):
        kv.append(K[t], V[t])
    kv.enable_page_summaries(page)
    c = Cache(L, Hkv, D, p0 + 64, page_size=128)
    c.append(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    c.enable_page_summaries(page)
    r = Runner(c, Hq, max_rows=5, max_prefix=p0, sparse_ratio=0.1, k_min=16)
    r.set_batch([0], [p0])
    q = normal_bf16(9, 1, (1, Hq, D))
    r.select_quest(1, to_dev_bf16(q))
    idx, cnt = r.selection(1, 1)
    want = kv.select_quest(q[0], 1, p0, 0.1, 16)
    assert cnt[0, 0] == selection_k(0.1, p0, 16) == len(want)
    assert np.array_equal(idx[0, 0, : cnt[0, 0]], want)
    c.close()


# ------------------------------------------------------------------- full-size cases (BASELINE configs)

def _bf16_round(x):
    """float32 -> nearest-even bf16-representable float32 (the device stores these bits losslessly)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    u = (u + (0x7FFF + ((u >> 16) & 1))) & 0xFFFF0000
    return u.view(np.float32)


FULL_CASES = [
    # (Hkv, G, R, p0, k)   k = None: selection_k(0.07, p0, 16) as in configs 2-4
    (8, 4, 5, 32768, None),   # config 2: one Llama-3.1-8B layer at 32K, gamma 4, k = 2294
    (1, 8, 5, 131072, None),  # config 4 per-GPU shard: one KV head (+ its 8 q-heads) at 128K, k = 9175
    (8, 4, 9, 32768, 4096),   # config 5 corner: gamma 8, k 4096
    (8, 4, 3, 32768, 64),     # config 5 corner: gamma 2, k 64
    (8, 4, 9, 32768, 2300),   # k + tail crosses 12 x 192 rows mid-chain: single-round drafts with 13-CTA clusters
]


@pytest.mark.parametrize("Hkv,G,R,p0,kfix", FULL_CASES)
def test_full_size_verify_select_draft(cuda, ref, Hkv, G, R, p0, kfix):
    """One layer at the BASELINE configs' full context: verify (outputs + fused Collect-2 scores),
    per-layer top-k and the gamma draft steps over the selected rows, each against the reference's own
    CPU code (oracle/_ref) on the same bf16-representable inputs (numpy Philox, not CounterRng, to keep
    the 10^8-element generation fast; the parity contract is on identical inputs either way)."""
    torch = cuda
    Runner, _, selection_k = _lib()
    from paper_2602_07223_b200 import Cache
    rng = np.random.default_rng(p0 + 97 * R + Hkv)
    Hq = Hkv * G
    ratio, k_min = (1e-9, kfix) if kfix else (0.07, 16)
    k = selection_k(ratio, p0, k_min)
    K = _bf16_round(rng.standard_normal((p0, Hkv, D), np.float32))
    V = _bf16_round(rng.standard_normal((p0, Hkv, D), np.float32))
    cache = Cache(1, Hkv, D, p0 + R + 64, page_size=256)
    for c0 in range(0, p0, 8192):
        cache.append(torch.from_numpy(K[c0:c0 + 8192]).cuda(), torch.from_numpy(V[c0:c0 + 8192]).cuda())
    kv = ref.kv(1, Hkv, D, p0 + R + 64)
    for t in range(p0):
        kv.append(K[t], V[t])
    r = Runner(cache, Hq, max_rows=R, max_prefix=p0, sparse_ratio=ratio, k_min=k_min)
    r.set_batch([0], [p0])
    q = _bf16_round(rng.standard_normal((1, Hq, R, D), np.float32))
    kn = _bf16_round(rng.standard_normal((1, R, Hkv, D), np.float32))
    vn = _bf16_round(rng.standard_normal((1, R, Hkv, D), np.float32))
    out = torch.zeros((1, Hq, R, D), dtype=torch.float32, device="cuda")
    r.verify(0, to_dev_bf16(q), out, to_dev_bf16(kn), to_dev_bf16(vn), SCALE, score_row_mask=1 | (1 << (R - 1)))
    idx, cnt = _gpu_select(r, 0, 0, 1, 2)
    for t in range(R):
        kv.append(kn[0, t], vn[0, t])
    o_ref, l_ref = kv.verify_layer(0, Hq, q[0], p0, R, SCALE, threads=8)
    got = out.cpu().numpy()[0]
    assert rel_err_rows(got, o_ref) < 2e-4, rel_err_rows(got, o_ref)
    assert rel_err_elem(got, o_ref) < 2e-3
    # selection: |T| = k, bit-exact outside the 2e-3 tie band (north star)
    ref_scores = ref.score_columns(l_ref, list(range(1, R + 1)), [1, R])
    assert cnt[0, 0] == k
    sel = idx[0, 0, :k].astype(np.int64)
    check_selection(sel, ref_scores, k)
    # draft chain over the GPU's selection (drafts read T; parity of attention given T)
    kv.truncate(p0)
    cache.set_size(p0)
    for step in range(1, R):
        qd = _bf16_round(rng.standard_normal((1, Hq, D), np.float32))
        kd = _bf16_round(rng.standard_normal((1, Hkv, D), np.float32))
        vd = _bf16_round(rng.standard_normal((1, Hkv, D), np.float32))
        o = torch.zeros((1, Hq, D), dtype=torch.float32, device="cuda")
        r.draft(0, step, to_dev_bf16(qd), o, to_dev_bf16(kd), to_dev_bf16(vd), mode=0, scale=SCALE)
        kv.append(kd[0], vd[0])
        o_ref = kv.draft_layer(0, Hq, qd[0], [sel], p0, step, SCALE, threads=8)
        got = o.cpu().numpy()[0]
        assert rel_err_rows(got, o_ref) < 2e-4, (step, rel_err_rows(got, o_ref))
        assert rel_err_elem(got, o_ref) < 2e-3
