"""ctypes bindings for the CPU checkers — TEST INFRASTRUCTURE ONLY.

`Oracle` wraps oracle/build/liboracle.so (the plain-C restatement); `Ref` wraps
oracle/_ref/libspecattn_ref.so (the reference's own TUs compiled against the
Eigen shim).  Both expose the same numpy-level methods so tests can run every
known-answer check against both and compare them bit-for-bit.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
reference) may import this module; the product path never does.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspecattn_ref.so")

STATUS_EXC = {1: ValueError, 2: ArithmeticError, 3: IndexError, 4: OverflowError}
STATUS_NAME = {0: "ok", 1: "invalid_argument", 2: "domain_error", 3: "out_of_range", 4: "length_error"}

# selection.hpp:15-22 numbering used by both C entry points
LAST_ACCEPTED, ALL_DRAFT, COLLECT2, COLLECT2_WEIGHTS = 2, 3, 4, 5


class OracleError(Exception):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {STATUS_NAME.get(status, status)}")
        self.status = status


def _check(st: int, what: str) -> None:
    if st != 0:
        raise OracleError(st, what)


_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64 = C.c_int64
_vp = C.c_void_p


def _nullable(a, dtype):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype).ctypes.data_as(_vp)


def build(ref: bool = True) -> None:
    """Build the checker libraries (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"] + (["ref"] if ref else []), check=True)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class _Base:
    lib: C.CDLL

    # ---- attention ----
    def softmax_stable(self, logits, scale=1.0):
        logits = _f32(logits)
        out = np.empty(logits.size, np.float64)
        _check(self._softmax(logits, logits.size, float(scale), out), "softmax_stable")
        return out

    def attend(self, q, K, V, scale):
        q, K, V = _f32(q), _f32(K).reshape(-1, q.size), _f32(V).reshape(-1, q.size)
        out = np.empty(q.size, np.float32)
        _check(self._attend(q, K, V, K.shape[0], q.size, float(scale), out), "attend")
        return out

    def attend_collect(self, q, Kp, Vp, Kw, Vw, scale):
        d = np.size(q)
        q = _f32(q)
        Kp, Vp = _f32(Kp).reshape(-1, d), _f32(Vp).reshape(-1, d)
        Kw, Vw = _f32(Kw).reshape(-1, d), _f32(Vw).reshape(-1, d)
        out = np.empty(d, np.float32)
        logits = np.empty(max(Kp.shape[0], 1), np.float32)
        _check(self._attend_collect(q, Kp, Vp, Kp.shape[0], Kw, Vw, Kw.shape[0], d, float(scale), out, logits),
               "attend_collect")
        return out, logits[: Kp.shape[0]]

    # ---- selection ----
    def selection_k(self, ratio, p, k_min):
        return int(self._selection_k(float(ratio), int(p), int(k_min)))

    def topk_indices(self, scores, k):
        scores = np.ascontiguousarray(scores, np.float64)
        out = np.empty(max(int(k), 1), np.int64)
        n = _i64(0)
        _check(self._topk(scores, scores.size, int(k), out, C.byref(n)), "topk_indices")
        return out[: n.value].copy()

    def score_columns(self, L, row_labels, sel, weights=False, head_dim=0):
        L = _f32(L)
        H, R, Cc = L.shape
        labels = np.ascontiguousarray(row_labels, np.int32)
        sel = np.ascontiguousarray(sel, np.int32)
        out = np.empty(max(Cc, 1), np.float64)
        _check(self._score(L, H, R, Cc, labels, sel, sel.size, int(weights), int(head_dim), out), "score_columns")
        return out[:Cc]

    def select(self, strategy, L, row_labels, ratio, k_min, accepted=0, head_dim=128):
        L = _f32(L)
        H, R, Cc = L.shape
        labels = np.ascontiguousarray(row_labels, np.int32)
        out = np.empty(max(Cc, 1), np.int64)
        n = _i64(0)
        _check(self._select(int(strategy), L, H, R, Cc, labels, int(head_dim), float(ratio), int(k_min),
                            int(accepted), out, C.byref(n)), "select")
        return out[: n.value].copy()


class Oracle(_Base):
    """Plain-C restatement (oracle/specattn_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        self.lib = lib = C.CDLL(path)
        lib.so_softmax_stable.argtypes = [_f32p, _i64, C.c_double, _f64p]
        lib.so_attend.argtypes = [_f32p, _i64, _f32p, _f32p, _i64, C.c_float, _f32p]
        lib.so_attend_collect.argtypes = [_f32p, _i64, _f32p, _f32p, _i64, _f32p, _f32p, _i64, C.c_float, _f32p,
                                          _f32p]
        lib.so_selection_k.restype = _i64
        lib.so_selection_k.argtypes = [C.c_double, _i64, _i64]
        lib.so_topk_indices.argtypes = [_f64p, _i64, _i64, _i64p, C.POINTER(_i64)]
        lib.so_score_columns.argtypes = [_vp, _i32p, _i64, _f64p]
        lib.so_score_columns_weights.argtypes = [_vp, _i32p, _i64, _f64p]
        lib.so_select.argtypes = [C.c_int, _vp, C.c_double, _i64, C.c_int, _i64p, C.POINTER(_i64)]
        lib.so_kv_create.restype = _vp
        lib.so_kv_create.argtypes = [_i64, _i64, _i64, _i64]
        lib.so_kv_destroy.argtypes = [_vp]
        for f in ("so_kv_size", "so_kv_committed"):
            getattr(lib, f).restype = _i64
            getattr(lib, f).argtypes = [_vp]
        lib.so_kv_append.argtypes = [_vp, _f32p, _f32p]
        lib.so_kv_truncate.argtypes = [_vp, _i64]
        lib.so_kv_set_committed.argtypes = [_vp, _i64]
        lib.so_kv_gather.argtypes = [_vp, _i64, _i64, _i64p, _i64, _f32p, _f32p]
        lib.so_verify_layer.argtypes = [_vp, _i64, _i64, _f32p, _i64, _i64, C.c_float, _f32p, _vp]
        lib.so_draft_layer.argtypes = [_vp, _i64, _i64, _f32p, _i64p, _i64p, _i64, _i64, _i64, _i64, C.c_float,
                                       _f32p]
        lib.so_rng_mix64.restype = C.c_uint64
        lib.so_rng_mix64.argtypes = [C.c_uint64]
        lib.so_rng_seeded_key.restype = C.c_uint64
        lib.so_rng_seeded_key.argtypes = [C.c_uint64]
        lib.so_rng_derive_key.restype = C.c_uint64
        lib.so_rng_derive_key.argtypes = [C.c_uint64, C.c_uint64]
        lib.so_rng_at.restype = C.c_uint64
        lib.so_rng_at.argtypes = [C.c_uint64, C.c_uint64]
        lib.so_rng_normals.argtypes = [C.c_uint64, _i64, _f64p]

    def _softmax(self, *a):
        return self.lib.so_softmax_stable(a[0], a[1], a[2], a[3])

    def _attend(self, q, K, V, m, d, scale, out):
        return self.lib.so_attend(q, d, K, V, m, scale, out)

    def _attend_collect(self, q, Kp, Vp, m0, Kw, Vw, m1, d, scale, out, logits):
        return self.lib.so_attend_collect(q, d, Kp, Vp, m0, Kw, Vw, m1, scale, out, logits)

    def _selection_k(self, *a):
        return self.lib.so_selection_k(*a)

    def _topk(self, *a):
        return self.lib.so_topk_indices(*a)

    class _LM(C.Structure):
        _fields_ = [("logits", _vp), ("n_heads", _i64), ("rows", _i64), ("cols", _i64), ("row_labels", _vp),
                    ("head_dim", _i64), ("layer", _i64)]

    def _lm(self, L, H, R, Cc, labels, head_dim):
        return self._LM(L.ctypes.data_as(_vp), H, R, Cc, labels.ctypes.data_as(_vp), head_dim, 0)

    def _score(self, L, H, R, Cc, labels, sel, nsel, weights, head_dim, out):
        lm = self._lm(L, H, R, Cc, labels, head_dim)
        f = self.lib.so_score_columns_weights if weights else self.lib.so_score_columns
        return f(C.byref(lm), sel, nsel, out)

    def _select(self, strategy, L, H, R, Cc, labels, head_dim, ratio, k_min, accepted, out, n):
        lm = self._lm(L, H, R, Cc, labels, head_dim)
        return self.lib.so_select(strategy, C.byref(lm), ratio, k_min, accepted, out, n)

    def kv(self, n_layers, n_kv_heads, head_dim, max_context):
        return KvHandle(self, n_layers, n_kv_heads, head_dim, max_context)

    # rng.hpp
    def rng_seeded_key(self, seed):
        return int(self.lib.so_rng_seeded_key(seed))

    def rng_derive_key(self, key, label):
        return int(self.lib.so_rng_derive_key(key, label))

    def rng_at(self, key, i):
        return int(self.lib.so_rng_at(key, i))

    def rng_normals(self, key, n):
        out = np.empty(n, np.float64)
        self.lib.so_rng_normals(key, n, out)
        return out


class Ref(_Base):
    """The reference's own TUs (oracle/_ref/libspecattn_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle ref; needs /root/reference)")
        self.lib = lib = C.CDLL(path)
        lib.ref_softmax_stable.argtypes = [_f32p, _i64, C.c_double, _f64p]
        lib.ref_attend.argtypes = [_f32p, _f32p, _f32p, _i64, _i64, C.c_float, _f32p]
        lib.ref_attend_collect.argtypes = [_f32p, _f32p, _f32p, _i64, _f32p, _f32p, _i64, _i64, C.c_float, _f32p,
                                           _f32p]
        lib.ref_selection_k.restype = _i64
        lib.ref_selection_k.argtypes = [C.c_double, _i64, _i64]
        lib.ref_topk_indices.argtypes = [_f64p, _i64, _i64, _i64p, C.POINTER(_i64)]
        lib.ref_score_columns.argtypes = [_f32p, _i64, _i64, _i64, _i32p, _i32p, _i64, C.c_int, _i64, _f64p]
        lib.ref_select.argtypes = [C.c_int, _f32p, _i64, _i64, _i64, _i32p, _i64, C.c_double, _i64, C.c_int, _i64p,
                                   C.POINTER(_i64)]
        lib.ref_kv_create.restype = _vp
        lib.ref_kv_create.argtypes = [_i64, _i64, _i64, _i64]
        lib.ref_kv_destroy.argtypes = [_vp]
        for f in ("ref_kv_size", "ref_kv_committed", "ref_kv_bytes_per_token"):
            getattr(lib, f).restype = _i64
            getattr(lib, f).argtypes = [_vp]
        lib.ref_kv_append.argtypes = [_vp, _f32p, _f32p]
        lib.ref_kv_truncate.argtypes = [_vp, _i64]
        lib.ref_kv_set_committed.argtypes = [_vp, _i64]
        lib.ref_kv_gather.argtypes = [_vp, _i64, _i64, _i64p, _i64, _f32p, _f32p]
        lib.ref_kv_rows.argtypes = [_vp, _i64, _i64, _i64, _i64, _f32p, _f32p]
        lib.ref_kv_enable_page_summaries.argtypes = [_vp, _i64]
        lib.ref_kv_page_minmax.argtypes = [_vp, _i64, _i64, _f32p, _f32p, C.POINTER(_i64)]
        lib.ref_select_quest.argtypes = [_vp, _f32p, _i64, _i64, _i64, C.c_double, _i64, _i64p, C.POINTER(_i64)]
        lib.ref_select_window.argtypes = [_i64, _i64, _i64, _i64p, C.POINTER(_i64)]
        lib.ref_verify_layer.argtypes = [_vp, _i64, _i64, _f32p, _i64, _i64, C.c_float, _f32p, _vp, C.c_int]
        lib.ref_draft_layer.argtypes = [_vp, _i64, _i64, _f32p, _i64p, _i64p, _i64, _i64, _i64, _i64, C.c_float,
                                        _f32p, C.c_int]

    def _softmax(self, *a):
        return self.lib.ref_softmax_stable(*a)

    def _attend(self, *a):
        return self.lib.ref_attend(*a)

    def _attend_collect(self, *a):
        return self.lib.ref_attend_collect(*a)

    def _selection_k(self, *a):
        return self.lib.ref_selection_k(*a)

    def _topk(self, *a):
        return self.lib.ref_topk_indices(*a)

    def _score(self, *a):
        return self.lib.ref_score_columns(*a)

    def _select(self, *a):
        return self.lib.ref_select(*a)

    def kv(self, n_layers, n_kv_heads, head_dim, max_context):
        return KvHandle(self, n_layers, n_kv_heads, head_dim, max_context)


class KvHandle:
    """KvStore over either backend; numpy in/out."""

    def __init__(self, backend: _Base, n_layers, n_kv_heads, head_dim, max_context):
        self.b = backend
        self.L, self.Hkv, self.d, self.max_context = n_layers, n_kv_heads, head_dim, max_context
        self.is_ref = isinstance(backend, Ref)
        p = "ref_kv_" if self.is_ref else "so_kv_"
        self._f = lambda name: getattr(backend.lib, p + name)
        self.h = self._f("create")(n_layers, n_kv_heads, head_dim, max_context)

    def __del__(self):
        if getattr(self, "h", None):
            self._f("destroy")(self.h)
            self.h = None

    def size(self):
        return int(self._f("size")(self.h))

    def committed(self):
        return int(self._f("committed")(self.h))

    def append(self, keys, values):
        keys = _f32(keys).reshape(self.L * self.Hkv, self.d)
        values = _f32(values).reshape(self.L * self.Hkv, self.d)
        _check(self._f("append")(self.h, keys, values), "append")
        return self.size()

    def truncate(self, n):
        _check(self._f("truncate")(self.h, int(n)), "truncate")

    def set_committed(self, n):
        _check(self._f("set_committed")(self.h, int(n)), "set_committed")

    def gather(self, layer, head, idx):
        idx = np.ascontiguousarray(idx, np.int64)
        K = np.empty((max(idx.size, 1), self.d), np.float32)
        V = np.empty_like(K)
        _check(self._f("gather")(self.h, int(layer), int(head), idx, idx.size, K, V), "gather")
        return K[: idx.size].copy(), V[: idx.size].copy()

    def rows(self, layer, head, begin, n):
        if self.is_ref:
            K = np.empty((max(n, 1), self.d), np.float32)
            V = np.empty_like(K)
            _check(self.b.lib.ref_kv_rows(self.h, layer, head, begin, n, K, V), "rows")
            return K[:n].copy(), V[:n].copy()
        return self.gather(layer, head, np.arange(begin, begin + n))

    # ---- Quest page summaries / baseline selectors (reference backend: the reference's own code)
    def enable_page_summaries(self, page_size):
        _check(self.b.lib.ref_kv_enable_page_summaries(self.h, int(page_size)), "enable_page_summaries")
        self.page_size = int(page_size)

    def page_minmax(self, layer, head):
        n_max = (self.size() + self.page_size - 1) // self.page_size
        mn = np.empty((max(n_max, 1), self.d), np.float32)
        mx = np.empty_like(mn)
        n = _i64(0)
        _check(self.b.lib.ref_kv_page_minmax(self.h, layer, head, mn, mx, C.byref(n)), "page_minmax")
        return mn[: n.value].copy(), mx[: n.value].copy()

    def select_quest(self, q_heads, layer, prefix_len, ratio, k_min):
        q = _f32(q_heads).reshape(-1, self.d)
        out = np.empty(max(prefix_len, 1), np.int64)
        n = _i64(0)
        _check(self.b.lib.ref_select_quest(self.h, q, q.shape[0], layer, prefix_len, float(ratio), int(k_min), out,
                                           C.byref(n)), "select_quest")
        return out[: n.value].copy()

    def verify_layer(self, layer, n_q_heads, q, p0, R, scale, want_logits=True, threads=1):
        q = _f32(q).reshape(n_q_heads, R, self.d)
        out = np.empty((n_q_heads, R, self.d), np.float32)
        logits = np.empty((n_q_heads, R, max(p0, 1)), np.float32) if want_logits else None
        lp = None if logits is None else logits.ctypes.data_as(_vp)
        if self.is_ref:
            st = self.b.lib.ref_verify_layer(self.h, layer, n_q_heads, q, p0, R, float(scale), out, lp, threads)
        else:
            st = self.b.lib.so_verify_layer(self.h, layer, n_q_heads, q, p0, R, float(scale), out, lp)
        _check(st, "verify_layer")
        return out, (None if logits is None else logits[:, :, :p0].copy())

    def draft_layer(self, layer, n_q_heads, q, idx_sets, tail_begin, tail_len, scale, threads=1):
        """idx_sets: list of 1 (per-layer) or Hkv (per-kv-head) ascending index arrays."""
        q = _f32(q).reshape(n_q_heads, self.d)
        n_sets = len(idx_sets)
        ks = np.array([len(s) for s in idx_sets], np.int64)
        stride = max(int(ks.max()) if n_sets else 1, 1)
        idx = np.zeros((n_sets, stride), np.int64)
        for i, s in enumerate(idx_sets):
            idx[i, : len(s)] = s
        out = np.empty((n_q_heads, self.d), np.float32)
        if self.is_ref:
            st = self.b.lib.ref_draft_layer(self.h, layer, n_q_heads, q, idx, ks, n_sets, stride, tail_begin,
                                            tail_len, float(scale), out, threads)
        else:
            st = self.b.lib.so_draft_layer(self.h, layer, n_q_heads, q, idx, ks, n_sets, stride, tail_begin,
                                           tail_len, float(scale), out)
        _check(st, "draft_layer")
        return out


def ref_select_window(ref, prefix_len, sink, window):
    """select_window (selection.cpp:209-222) from the reference's own code."""
    out = np.empty(max(prefix_len, 1), np.int64)
    n = _i64(0)
    _check(ref.lib.ref_select_window(int(prefix_len), int(sink), int(window), out, C.byref(n)), "select_window")
    return out[: n.value].copy()


def quest_bounds(mins, maxs, q_heads, group):
    """Restatement of select_quest's page upper bounds (selection.cpp:237-248): per q-head h (KV head
    h // group) the float sum over d of max(q*min, q*max), accumulated over heads in double.
    mins/maxs: [Hkv][n_pages][d] f32, q_heads: [Hq][d] f32 -> [n_pages] f64."""
    q = np.asarray(q_heads, np.float32)
    b = np.zeros(mins.shape[1], np.float64)
    for h in range(q.shape[0]):
        g = h // group
        t = np.maximum(q[h] * mins[g], q[h] * maxs[g]).astype(np.float32)
        b += t.sum(axis=1, dtype=np.float32).astype(np.float64)
    return b


def quest_pick(bounds, prefix_len, page, k):
    """Restatement of select_quest's page ordering and token pick (selection.cpp:250-271)."""
    order = sorted(range(len(bounds)), key=lambda p: (-bounds[p], p))
    picked = []
    for p in order:
        if len(picked) >= k:
            break
        for i in range(p * page, min(p * page + page, prefix_len)):
            if len(picked) >= k:
                break
            picked.append(i)
    return np.array(sorted(picked), np.int64)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 to the nearest bf16 (RNE) and return as fp32 (exactly representable)."""
    x = np.ascontiguousarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    out = r.astype(np.uint32).view(np.float32)
    return np.where(np.isnan(x), x, out)


def scale_for(head_dim: int) -> float:
    """float(1/sqrt(d)) as used on both sides."""
    return float(np.float32(1.0 / math.sqrt(head_dim)))
