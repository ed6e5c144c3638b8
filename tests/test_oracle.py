"""CPU tests: pin the C restatement (oracle/) against the reference's own code and the SPEC
known-answer tests, plus the committed golden vectors (tests/golden/)."""
import itertools
import math
import os

import numpy as np
import pytest

from oracle.counter_rng import CounterRng, normal_bf16
from oracle.pyoracle import ALL_DRAFT, COLLECT2, COLLECT2_WEIGHTS, LAST_ACCEPTED, OracleError, scale_for

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz")


@pytest.fixture(params=["oracle", "ref"])
def impl(request, oracle):
    if request.param == "oracle":
        return oracle
    return request.getfixturevalue("ref")


# ----------------------------------------------------------------- rng (rng.hpp)

def test_counter_rng_kats(oracle):
    # values recorded in SURVEY.md §8c from the reference header compiled standalone
    assert CounterRng.seeded(7).at(0) == 5552335213642010640
    assert oracle.rng_at(oracle.rng_seeded_key(7), 0) == 5552335213642010640
    v = CounterRng.seeded(7).derive(3).normals(1)[0]
    assert v == pytest.approx(-0.45698742437892576, abs=1e-15)
    key = CounterRng.seeded(11).derive(5).key
    assert np.allclose(CounterRng(key).normals(64), oracle.rng_normals(key, 64), rtol=0, atol=1e-15)


# ----------------------------------------------------------------- attention

def test_softmax_kats(impl):
    assert np.array_equal(impl.softmax_stable([0.0, 0.0]), [0.5, 0.5])
    assert np.array_equal(impl.softmax_stable([3.25]), [1.0])
    rng = np.random.default_rng(0)
    v = rng.standard_normal(33).astype(np.float32)
    a, b = impl.softmax_stable(v), impl.softmax_stable(v + np.float32(4.0))
    assert np.max(np.abs(a - b)) < 1e-6  # shift invariance (float shift, double softmax)
    assert abs(a.sum() - 1.0) < 1e-9
    masked = impl.softmax_stable(np.array([1.0, -np.inf, 2.0], np.float32))
    assert masked[1] == 0.0
    with pytest.raises(OracleError) as e:
        impl.softmax_stable(np.array([-np.inf, -np.inf], np.float32))
    assert e.value.status == 2  # std::domain_error
    with pytest.raises(OracleError) as e:
        impl.softmax_stable([1.0], scale=0.0)
    assert e.value.status == 1


def test_attend_kats(impl):
    rng = np.random.default_rng(1)
    d = 4
    q = rng.standard_normal(d).astype(np.float32)
    V = rng.standard_normal((1, d)).astype(np.float32)
    assert np.array_equal(impl.attend(q, rng.standard_normal((1, d)), V, 0.5), V[0])  # m=1 -> V[0]
    K = np.tile(rng.standard_normal((1, d)).astype(np.float32), (5, 1))
    V = rng.standard_normal((5, d)).astype(np.float32)
    assert np.allclose(impl.attend(q, K, V, 0.5), V.astype(np.float64).mean(0), rtol=1e-6, atol=1e-7)
    # random m=8, d=4 vs an fp64 naive loop, 1e-5 relative
    K = rng.standard_normal((8, d)).astype(np.float32)
    V = rng.standard_normal((8, d)).astype(np.float32)
    lg = K.astype(np.float64) @ q.astype(np.float64) * 0.5
    w = np.exp(lg - lg.max())
    w /= w.sum()
    assert np.allclose(impl.attend(q, K, V, 0.5), w @ V.astype(np.float64), rtol=1e-5, atol=1e-6)
    with pytest.raises(OracleError) as e:
        impl.attend(q, np.zeros((0, d)), np.zeros((0, d)), 0.5)
    assert e.value.status == 1


def test_attend_collect_kats(impl):
    rng = np.random.default_rng(2)
    d = 128
    q = normal_bf16(3, 1, (d,))
    Kp, Vp = normal_bf16(3, 2, (40, d)), normal_bf16(3, 3, (40, d))
    Kw, Vw = normal_bf16(3, 4, (3, d)), normal_bf16(3, 5, (3, d))
    s = scale_for(d)
    out, logits = impl.attend_collect(q, Kp, Vp, Kw, Vw, s)
    full = impl.attend(q, np.concatenate([Kp, Kw]), np.concatenate([Vp, Vw]), s)
    assert np.array_equal(out, full)  # == attend(concat), bitwise here
    naive = Kp.astype(np.float64) @ q.astype(np.float64)
    assert np.allclose(logits, naive, rtol=1e-5, atol=1e-5 * np.abs(Kp * q).sum(1).max())
    out0, lg0 = impl.attend_collect(q, np.zeros((0, d)), np.zeros((0, d)), Kw, Vw, s)  # empty prefix
    assert lg0.size == 0 and np.array_equal(out0, impl.attend(q, Kw, Vw, s))
    del rng


# ----------------------------------------------------------------- selection

def test_topk_kats(impl):
    assert list(impl.topk_indices([5, 1, 5, 0], 2)) == [0, 2]
    assert list(impl.topk_indices([3, 2, 1], 3)) == [0, 1, 2]
    assert list(impl.topk_indices([1.0, -np.inf, 2.0], 3)) == [0, 2]  # -inf never selected
    with pytest.raises(OracleError):
        impl.topk_indices([1.0, 2.0], 3)


def test_topk_matches_exhaustive_subset(impl):
    """AC3: top-k of column sums == argmax over all C(p,k) subsets, lower-index ties."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        p = int(rng.integers(1, 13))
        k = int(rng.integers(0, min(4, p) + 1))
        s = rng.integers(-3, 4, p).astype(np.float64)  # small ints -> frequent ties
        best, best_key = None, None
        for sub in itertools.combinations(range(p), k):
            key = (sum(s[list(sub)]), [-i for i in sub])  # larger sum, then lexicographically smaller
            if best_key is None or key > best_key:
                best_key, best = key, list(sub)
        assert list(impl.topk_indices(s, k)) == best


def test_selection_k_kats(impl):
    assert impl.selection_k(0.25, 100, 16) == 25
    assert impl.selection_k(0.01, 100, 16) == 16
    assert impl.selection_k(0.5, 10, 16) == 10
    assert impl.selection_k(0.07, 32768, 16) == 2294
    assert impl.selection_k(0.07, 65536, 16) == 4588
    assert impl.selection_k(0.07, 131072, 16) == 9175


def test_score_columns_kats(impl):
    rng = np.random.default_rng(4)
    L = rng.standard_normal((1, 1, 9)).astype(np.float32)
    assert np.array_equal(impl.score_columns(L, [1], [1]), L[0, 0].astype(np.float64))
    L2 = np.repeat(L, 2, axis=1)
    assert np.array_equal(impl.score_columns(L2, [1, 2], [1, 2]), L[0, 0].astype(np.float64))
    L3 = rng.standard_normal((2, 3, 7)).astype(np.float32)
    want = np.array([sum(float(L3[h, r, c]) for h in range(2) for r in (0, 2)) / 4 for c in range(7)])
    assert np.array_equal(impl.score_columns(L3, [1, 2, 3], [1, 3]), want)
    with pytest.raises(OracleError):
        impl.score_columns(L3, [1, 2, 3], [])
    with pytest.raises(OracleError):
        impl.score_columns(L3, [1, 2, 3], [4])
    Lw = np.zeros((1, 1, 4), np.float32)
    assert np.allclose(impl.score_columns(Lw, [1], [1], weights=True, head_dim=128), 0.25)


def test_select_strategies(impl):
    rng = np.random.default_rng(5)
    L = rng.standard_normal((4, 5, 60)).astype(np.float32)
    labels = [1, 2, 3, 4, 5]
    c2 = impl.select(COLLECT2, L, labels, 0.25, 4)
    rows = impl.select(ALL_DRAFT, L[:, [0, 4], :], [1, 5], 0.25, 4)
    assert np.array_equal(c2, rows)  # Collect-2 == AllDraft restricted to {1, gamma+1}
    assert len(c2) == impl.selection_k(0.25, 60, 4)
    assert np.all(np.diff(c2) > 0)
    la = impl.select(LAST_ACCEPTED, L, labels, 0.25, 4, accepted=0)
    assert np.array_equal(la, impl.select(ALL_DRAFT, L[:, :1, :], [1], 0.25, 4))
    same = np.repeat(L[:, :1, :], 5, axis=1)
    assert np.array_equal(impl.select(COLLECT2, same, labels, 0.25, 4), impl.select(ALL_DRAFT, same, labels, 0.25, 4))
    impl.select(COLLECT2_WEIGHTS, L, labels, 0.25, 4)
    with pytest.raises(OracleError):
        impl.select(LAST_ACCEPTED, L, labels, 0.25, 4, accepted=5)
    # scale invariance x3.7 (AC7) and monotone k
    for s in (COLLECT2, ALL_DRAFT):
        assert np.array_equal(impl.select(s, L, labels, 0.25, 4), impl.select(s, L * np.float32(3.7), labels, 0.25, 4))
    sc = impl.score_columns(L, labels, [1, 5])
    for k in range(1, 59):
        assert set(impl.topk_indices(sc, k)) <= set(impl.topk_indices(sc, k + 1))


# ----------------------------------------------------------------- kv store

def test_kv_store_kats(impl):
    kv = impl.kv(2, 2, 8, 10)
    rng = np.random.default_rng(6)
    toks = [(rng.standard_normal((4, 8)).astype(np.float32), rng.standard_normal((4, 8)).astype(np.float32))
            for _ in range(6)]
    for k, v in toks[:5]:
        kv.append(k, v)
    kv.set_committed(4)
    kv.truncate(3)
    assert kv.committed() == 3
    assert kv.append(*toks[5]) == 4
    K, V = kv.gather(1, 1, [0, 3])
    assert np.array_equal(K[1], toks[5][0][3]) and np.array_equal(V[0], toks[0][1][3])
    with pytest.raises(OracleError) as e:
        kv.truncate(5)
    assert e.value.status == 3
    with pytest.raises(OracleError) as e:
        kv.gather(0, 0, [2, 1])
    assert e.value.status == 3
    with pytest.raises(OracleError) as e:
        kv.gather(0, 0, [4])
    assert e.value.status == 3
    assert kv.gather(0, 0, [])[0].shape == (0, 8)
    full = impl.kv(1, 1, 8, 2)
    full.append(toks[0][0][:1], toks[0][1][:1])
    full.append(toks[0][0][:1], toks[0][1][:1])
    with pytest.raises(OracleError) as e:
        full.append(toks[0][0][:1], toks[0][1][:1])
    assert e.value.status == 4  # std::length_error


def test_kv_bytes_kat(ref):
    kv = ref.kv(4, 2, 32, 16)
    assert int(ref.lib.ref_kv_bytes_per_token(kv.h)) == 2048  # SPEC.md:148 toy config


# ----------------------------------------------------------------- restatement == reference

def test_restatement_bitwise_matches_reference(oracle, ref):
    d, Hq, Hkv, L = 128, 8, 2, 2
    p0, R = 70, 3
    n_tok = p0 + R
    ko, kr = oracle.kv(L, Hkv, d, 256), ref.kv(L, Hkv, d, 256)
    K = normal_bf16(21, 1, (n_tok, L * Hkv, d))
    V = normal_bf16(21, 2, (n_tok, L * Hkv, d))
    for t in range(n_tok):
        ko.append(K[t], V[t])
        kr.append(K[t], V[t])
    q = normal_bf16(21, 3, (Hq, R, d))
    s = scale_for(d)
    for layer in range(L):
        oo, lo = ko.verify_layer(layer, Hq, q, p0, R, s)
        orr, lr = kr.verify_layer(layer, Hq, q, p0, R, s, threads=4)
        assert np.array_equal(oo, orr) and np.array_equal(lo, lr)
        sets = [np.array(sorted(np.random.default_rng(layer + g).choice(p0, 9, replace=False))) for g in range(Hkv)]
        qd = normal_bf16(21, 4, (Hq, d))
        assert np.array_equal(ko.draft_layer(layer, Hq, qd, sets, p0, 2, s), kr.draft_layer(layer, Hq, qd, sets, p0, 2, s))
        assert np.array_equal(ko.draft_layer(layer, Hq, qd, sets[:1], p0, 3, s),
                              kr.draft_layer(layer, Hq, qd, sets[:1], p0, 3, s, threads=2))
    rng = np.random.default_rng(7)
    for _ in range(20):
        Lm = rng.standard_normal((3, 4, 37)).astype(np.float32)
        for strat in (ALL_DRAFT, COLLECT2, COLLECT2_WEIGHTS, LAST_ACCEPTED):
            assert np.array_equal(oracle.select(strat, Lm, [1, 2, 3, 4], 0.3, 2, accepted=2),
                                  ref.select(strat, Lm, [1, 2, 3, 4], 0.3, 2, accepted=2))


# ----------------------------------------------------------------- golden vectors

def test_golden_vectors(oracle):
    """Outputs of the reference itself (oracle/_ref, tests/golden/make_golden.py) reproduced by the
    restatement without needing /root/reference at test time."""
    g = np.load(GOLDEN)
    s = float(g["scale"])
    out, lg = oracle.attend_collect(g["ac_q"], g["ac_Kp"], g["ac_Vp"], g["ac_Kw"], g["ac_Vw"], s)
    assert np.array_equal(out, g["ac_out"]) and np.array_equal(lg, g["ac_logits"])
    for i, strat in enumerate((ALL_DRAFT, COLLECT2, COLLECT2_WEIGHTS, LAST_ACCEPTED)):
        got = oracle.select(strat, g["sel_L"], list(range(1, g["sel_L"].shape[1] + 1)), 0.25, 4, accepted=2)
        assert np.array_equal(got, g[f"sel_{i}"][: int(g[f"sel_{i}_n"])])
    Lh, Hkv, d = (int(x) for x in g["vl_shape"])
    kv = oracle.kv(Lh, Hkv, d, 512)
    for t in range(g["vl_K"].shape[0]):
        kv.append(g["vl_K"][t], g["vl_V"][t])
    p0, R, Hq = int(g["vl_p0"]), int(g["vl_R"]), int(g["vl_Hq"])
    for layer in range(Lh):
        o, l = kv.verify_layer(layer, Hq, g["vl_q"], p0, R, s)
        assert np.array_equal(o, g[f"vl_out_{layer}"]) and np.array_equal(l, g[f"vl_logits_{layer}"])
        sets = [g[f"dr_set_{layer}_{h}"] for h in range(Hkv)]
        assert np.array_equal(kv.draft_layer(layer, Hq, g["dr_q"], sets, p0, 2, s), g[f"dr_out_{layer}"])
    assert math.isfinite(s)


# ----------------------------------------------------------------- Quest / window baselines

def test_window_and_quest_restatement_vs_reference(ref):
    """The Quest page bounds / pick restatement (oracle/pyoracle.py) against the reference's own
    select_quest, and select_window KATs (selection.cpp:209-274)."""
    from oracle.pyoracle import quest_bounds, quest_pick, ref_select_window
    assert ref_select_window(ref, 10, 4, 3).tolist() == [0, 1, 2, 3, 7, 8, 9]
    assert ref_select_window(ref, 5, 4, 3).tolist() == [0, 1, 2, 3, 4]
    assert ref_select_window(ref, 0, 4, 3).tolist() == []
    L, Hkv, d, page = 2, 2, 16, 8
    kv = ref.kv(L, Hkv, d, 512)
    K = normal_bf16(201, 1, (203, L * Hkv, d))
    for t in range(100):
        kv.append(K[t], K[t])
    kv.enable_page_summaries(page)
    for t in range(100, 203):  # summaries refreshed on append (refresh_tail_page)
        kv.append(K[t], K[t])
    for layer in range(L):
        mins = np.stack([kv.page_minmax(layer, g)[0] for g in range(Hkv)])
        maxs = np.stack([kv.page_minmax(layer, g)[1] for g in range(Hkv)])
        Kl = K[:, layer * Hkv:(layer + 1) * Hkv]
        for g in range(Hkv):
            for p_ in range(mins.shape[1]):
                blk = Kl[p_ * page:(p_ + 1) * page, g]
                assert np.array_equal(mins[g, p_], blk.min(0)) and np.array_equal(maxs[g, p_], blk.max(0))
        q = normal_bf16(202, layer, (4 * Hkv, d))
        for prefix in (203, 150, 57):
            want = kv.select_quest(q, layer, prefix, 0.3, 16)
            n_pages = (prefix + page - 1) // page
            b = quest_bounds(mins[:, :n_pages], maxs[:, :n_pages], q, 4)
            k = min(prefix, max(int(np.floor(0.3 * prefix + 0.5)), 16))
            assert np.array_equal(quest_pick(b, prefix, page, k), want)


# ----------------------------------------------------------------- speculation glue
# The reference ships no speculation code: the restatement (oracle/speculation.py) is pinned on the
# SPEC's own examples here and the GPU kernel on the restatement (tests/test_gpu_parity.py).

def test_residual_distribution_kats():
    from oracle.speculation import residual_distribution
    assert np.array_equal(residual_distribution([0.5, 0.5], [1.0, 0.0]), [0.0, 1.0])
    assert np.array_equal(residual_distribution([0.7, 0.3], [0.3, 0.7]), [1.0, 0.0])
    rng = np.random.default_rng(3)
    for _ in range(20):
        p, q = rng.dirichlet(np.ones(16)), rng.dirichlet(np.ones(16))
        r = residual_distribution(p, q)
        assert r.sum() == pytest.approx(1.0, abs=1e-12)
        assert np.all(r[p <= q] == 0.0)
    with pytest.raises(ValueError):
        residual_distribution([0.25, 0.75], [0.25, 0.75])


def test_accept_kats():
    from oracle.speculation import accept
    rng = np.random.default_rng(5)
    # q_t = p_t for all t -> every accept probability is 1; a = gamma
    for _ in range(20):
        p = rng.dirichlet(np.ones(32), size=5).astype(np.float32)
        draft = rng.integers(0, 32, size=4)
        a, em = accept(p, draft, q=p[:4], u=rng.random(5).astype(np.float32))
        assert a == 4 and em[:4] == list(draft) and len(em) == 5
    # vocab {a,b}: q = (1,0), p = (0.5,0.5): accept a w.p. 0.5, on reject emit b
    p = np.array([[0.5, 0.5], [0.5, 0.5]], np.float32)
    q = np.array([[1.0, 0.0]], np.float32)
    acc = 0
    for i in range(2000):
        a, em = accept(p, [0], q=q, u=np.array([rng.random(), rng.random()], np.float32))
        if a == 1:
            acc += 1
        else:
            assert em == [1]
    assert abs(acc / 2000 - 0.5) < 0.05
    # greedy: accept iff x_t = argmax p_t (ties -> lower id); corrected token = argmax
    p = np.array([[0.1, 0.45, 0.45], [0.6, 0.2, 0.2], [0.3, 0.3, 0.4]], np.float32)
    assert accept(p, [1, 0], greedy=True) == (2, [1, 0, 2])
    assert accept(p, [2, 0], greedy=True) == (0, [1])
    assert accept(p, [1, 2], greedy=True) == (1, [1, 0])


def test_accept_emission_matches_target():
    # single-step emission distribution equals p (modified rejection sampling is exact): Monte-Carlo
    from oracle.speculation import accept
    rng = np.random.default_rng(9)
    V = 4
    p = rng.dirichlet(np.ones(V), size=2).astype(np.float32)
    q = rng.dirichlet(np.ones(V), size=1).astype(np.float32)
    n = 6000
    counts = np.zeros(V)
    q64 = q[0].astype(np.float64)
    q64 /= q64.sum()
    for _ in range(n):
        x = rng.choice(V, p=q64)
        _, em = accept(p, [x], q=q, u=rng.random(2).astype(np.float32))
        counts[em[0]] += 1
    assert 0.5 * np.abs(counts / n - p[0]).sum() < 0.03


# ----------------------------------------------------------------- model-side producer

@pytest.mark.parametrize("style", [0, 1])
def test_apply_rope_kats(style):
    from oracle.model import apply_rope
    rng = np.random.default_rng(21 + style)
    v = rng.standard_normal(128)
    assert np.array_equal(apply_rope(v, 0, style=style), v)  # position 0 -> identity
    for pos in (1, 17, 4095, 131071):
        assert abs(np.linalg.norm(apply_rope(v, pos, style=style)) - np.linalg.norm(v)) <= 1e-6 * np.linalg.norm(v)
    for m, n in ((5, 3), (1000, 17), (40000, 39000)):  # relative-position identity
        q, k = rng.standard_normal(128), rng.standard_normal(128)
        lhs = apply_rope(q, m, style=style) @ apply_rope(k, n, style=style)
        rhs = apply_rope(q, m - n, style=style) @ k
        assert abs(lhs - rhs) <= 1e-5 * max(1.0, abs(rhs))
    with pytest.raises(ValueError):
        apply_rope(np.ones(7), 3)


def test_rms_norm_and_projection_shapes():
    from oracle.model import qkv_project, rms_norm
    x = np.array([[3.0, 4.0]])
    assert np.allclose(rms_norm(x, [1.0, 2.0], 0.0), [[3 / np.sqrt(12.5), 8 / np.sqrt(12.5)]])
    rng = np.random.default_rng(2)
    w = rng.standard_normal(((4 + 2 * 2) * 128, 64))
    q, k, v = qkv_project(rng.standard_normal((2, 3, 64)), w, np.ones(64), 4, 2, [0, 9])
    assert q.shape == (2, 4, 3, 128) and k.shape == (2, 3, 2, 128) and v.shape == (2, 3, 2, 128)
