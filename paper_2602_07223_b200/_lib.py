"""ctypes binding of include/specattn_b200.h (no torch types cross the ABI: plain pointers/sizes)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.environ.get("SA_LIB_PATH") or os.path.join(HERE, "lib", "libspecattn_b200.so")  # env: dev A/B only

SA_OK = 0
STATUS = {0: "ok", 1: "invalid_argument", 2: "domain_error", 3: "out_of_range", 4: "length_error",
          5: "cuda_error", 6: "not_supported", 7: "nccl_error"}
WINDOW, QUEST_LIKE, LAST_ACCEPTED, ALL_DRAFT, COLLECT2, COLLECT2_WEIGHTS = 0, 1, 2, 3, 4, 5
PER_LAYER, PER_KV_HEAD = 0, 1
PHASE_VERIFY, PHASE_SELECT, PHASE_DRAFT = 1, 2, 4
F32, BF16 = 0, 1


class SpecAttnError(RuntimeError):
    """Raised for any non-OK sa_status; .status carries the reference exception class name."""

    def __init__(self, status: int, message: str):
        self.status = STATUS.get(status, str(status))
        super().__init__(f"{self.status}: {message}")


_i64, _i32, _u32, _vp, _f32 = C.c_int64, C.c_int32, C.c_uint32, C.c_void_p, C.c_float


class CacheConfig(C.Structure):
    _fields_ = [("n_layers", _i64), ("n_kv_heads", _i64), ("head_dim", _i64), ("max_context", _i64),
                ("max_seqs", _i64), ("page_size", _i64), ("num_pages", _i64)]


class RunnerConfig(C.Structure):
    _fields_ = [("max_batch", _i32), ("n_q_heads", _i32), ("max_rows", _i32), ("max_prefix", _i64),
                ("sparse_ratio", C.c_double), ("k_min", _i64), ("n_layers_buf", _i32)]


class VerifyArgs(C.Structure):
    _fields_ = [("layer", _i32), ("layer_slot", _i32), ("n_rows", _i32), ("q", _vp), ("k_new", _vp),
                ("v_new", _vp), ("scale", _f32), ("score_row_mask", _u32), ("out", _vp), ("logits", _vp),
                ("ld_logits", _i64), ("collect_row_mask", _u32), ("score_layout", _i32)]


class SelectArgs(C.Structure):
    _fields_ = [("layer_slot", _i32), ("mode", C.c_int), ("rows_in_score", _i32)]


class DraftArgs(C.Structure):
    _fields_ = [("layer", _i32), ("layer_slot", _i32), ("mode", C.c_int), ("step", _i32), ("q", _vp),
                ("k_new", _vp), ("v_new", _vp), ("scale", _f32), ("out", _vp)]


class IterationArgs(C.Structure):
    _fields_ = [("gamma", _i32), ("strategy", C.c_int), ("mode", C.c_int), ("scale", _f32), ("qv", _vp),
                ("kv_new", _vp), ("vv_new", _vp), ("qd", _vp), ("kd_new", _vp), ("vd_new", _vp), ("out_v", _vp),
                ("out_d", _vp), ("use_graph", _i32), ("phases", _u32), ("accepted", _i32)]


# exported symbol -> (restype, argtypes)
SIGNATURES = {
    "sa_status_string": (C.c_char_p, [C.c_int]),
    "sa_last_error": (C.c_char_p, []),
    "sa_version": (C.c_char_p, []),
    "sa_selection_k": (_i64, [C.c_double, _i64, _i64]),
    "sa_cache_create": (C.c_int, [C.POINTER(CacheConfig), C.POINTER(_vp)]),
    "sa_cache_destroy": (C.c_int, [_vp]),
    "sa_kv_size": (C.c_int, [_vp, _i32, C.POINTER(_i64)]),
    "sa_kv_committed": (C.c_int, [_vp, _i32, C.POINTER(_i64)]),
    "sa_kv_bytes_per_token": (C.c_int, [_vp, C.POINTER(_i64), C.POINTER(_i64)]),
    "sa_kv_append": (C.c_int, [_vp, _i32, _i64, _vp, _vp, C.c_int, C.c_int, _vp]),
    "sa_kv_truncate": (C.c_int, [_vp, _i32, _i64]),
    "sa_kv_set_committed": (C.c_int, [_vp, _i32, _i64]),
    "sa_kv_reserve": (C.c_int, [_vp, _i32, _i64]),
    "sa_kv_set_size": (C.c_int, [_vp, _i32, _i64]),
    "sa_kv_gather": (C.c_int, [_vp, _i32, _i64, _i64, C.POINTER(_i64), _i64, _vp, _vp, _vp]),
    "sa_kv_read": (C.c_int, [_vp, _i32, _i64, _i64, _i64, _i64, _vp, _vp, _vp]),
    "sa_runner_create": (C.c_int, [_vp, C.POINTER(RunnerConfig), C.POINTER(_vp)]),
    "sa_runner_destroy": (C.c_int, [_vp]),
    "sa_runner_set_batch": (C.c_int, [_vp, _i32, C.POINTER(_i32), C.POINTER(_i64)]),
    "sa_runner_scores": (_vp, [_vp, _i32, C.POINTER(_i64)]),
    "sa_runner_layer_scores": (_vp, [_vp, _i32, C.POINTER(_i64)]),
    "sa_runner_indices": (_vp, [_vp, _i32, C.POINTER(_i32)]),
    "sa_runner_counts": (_vp, [_vp, _i32]),
    "sa_verify_attention": (C.c_int, [_vp, C.POINTER(VerifyArgs), _vp]),
    "sa_select_topk": (C.c_int, [_vp, C.POINTER(SelectArgs), _vp]),
    "sa_draft_attention": (C.c_int, [_vp, C.POINTER(DraftArgs), _vp]),
    "sa_iteration_run": (C.c_int, [_vp, C.POINTER(IterationArgs), _vp]),
    "sa_iteration_kernel_count": (_i64, [_vp, C.POINTER(IterationArgs)]),
    "sa_dev_trace_dump": (C.c_int, [_vp, C.c_char_p]),
    "sa_dev_set_knob": (C.c_int, [_vp, C.c_char_p, _i64]),
    "sa_qkv_dev_set_knob": (C.c_int, [_vp, C.c_char_p, _i64]),
    "sa_score_weights": (C.c_int, [_vp, _i32, _vp, _i64, _i32, C.c_int, _vp]),
    "sa_kv_enable_page_summaries": (C.c_int, [_vp, _i64]),
    "sa_qkv_create": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, C.c_double, C.c_double, _i32, C.POINTER(_vp)]),
    "sa_qkv_destroy": (C.c_int, [_vp]),
    "sa_qkv_project": (C.c_int, [_vp, _i32, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp]),
    "sa_accept": (C.c_int, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp]),
    "sa_kv_commit_accepted": (C.c_int, [_vp, _i32, _i64, _i32]),
    "sa_select_quest": (C.c_int, [_vp, _i32, _i32, _vp, _vp]),
    "sa_select_window": (C.c_int, [_vp, _i32, _i64, _i64, _vp]),
    "sa_comm_unique_id": (C.c_int, [_vp]),
    "sa_comm_create": (C.c_int, [_vp, _i32, _i32, C.POINTER(_vp)]),
    "sa_comm_destroy": (C.c_int, [_vp]),
    "sa_comm_info": (C.c_int, [_vp, C.POINTER(_i32), C.POINTER(_i32)]),
    "sa_comm_check": (C.c_int, [_vp]),
    "sa_comm_sync": (C.c_int, [_vp, _vp, _i64]),
    "sa_runner_set_comm": (C.c_int, [_vp, _vp]),
    "sa_exchange_layer_scores": (C.c_int, [_vp, _i32, _vp]),
}

_LIB = None


def build() -> None:
    """Compile the CUDA library in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    subprocess.run(["make", "-s", "-j8", "-C", os.path.join(HERE, "csrc")], check=True)


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not os.path.exists(lib_path):
            raise SpecAttnError(6, f"{lib_path} missing — run __graft_entry__.build(); there is no CPU fallback")
        L = C.CDLL(lib_path)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def _check(st: int) -> None:
    if st != SA_OK:
        raise SpecAttnError(st, lib().sa_last_error().decode())


def selection_k(ratio: float, p: int, k_min: int) -> int:
    return int(lib().sa_selection_k(ratio, p, k_min))


def _ptr(t) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise SpecAttnError(1, "device tensor expected")
    if not t.is_contiguous():
        raise SpecAttnError(1, "contiguous tensor expected")
    return t.data_ptr()


def _stream(stream) -> int | None:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class Cache:
    """Device KV store (sa_cache): the KvStore API of kv_store.hpp:19-89 over a paged bf16 pool."""

    def __init__(self, n_layers, n_kv_heads, head_dim=128, max_context=4096, max_seqs=1, page_size=256,
                 num_pages=0):
        import torch
        if not torch.cuda.is_available():
            raise SpecAttnError(5, "no CUDA device: the SpecAttn hot path has no CPU fallback")
        self.L, self.Hkv, self.d = n_layers, n_kv_heads, head_dim
        self.max_context, self.max_seqs = max_context, max_seqs
        cfg = CacheConfig(n_layers, n_kv_heads, head_dim, max_context, max_seqs, page_size, num_pages)
        h = _vp()
        _check(lib().sa_cache_create(C.byref(cfg), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().sa_cache_destroy(self.h)
            self.h = None

    __del__ = close

    def size(self, seq=0):
        n = _i64()
        _check(lib().sa_kv_size(self.h, seq, C.byref(n)))
        return n.value

    def committed(self, seq=0):
        n = _i64()
        _check(lib().sa_kv_committed(self.h, seq, C.byref(n)))
        return n.value

    def bytes_per_token(self):
        a, b = _i64(), _i64()
        _check(lib().sa_kv_bytes_per_token(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def append(self, keys, values, seq=0, stream=None):
        """keys/values: [n_tokens][L*Hkv][d] (or one token [L*Hkv][d]); fp32 or bf16, device or host."""
        import torch
        if keys.dim() == 2:
            keys, values = keys.unsqueeze(0), values.unsqueeze(0)
        keys, values = keys.contiguous(), values.contiguous()
        dt = F32 if keys.dtype == torch.float32 else BF16
        if keys.dtype not in (torch.float32, torch.bfloat16) or values.dtype != keys.dtype:
            raise SpecAttnError(1, "append expects fp32 or bf16")
        _check(lib().sa_kv_append(self.h, seq, keys.shape[0], keys.data_ptr(), values.data_ptr(), dt,
                                  0 if keys.is_cuda else 1, _stream(stream)))
        return self.size(seq)

    def truncate(self, to_len, seq=0):
        _check(lib().sa_kv_truncate(self.h, seq, to_len))

    def set_committed(self, n, seq=0):
        _check(lib().sa_kv_set_committed(self.h, seq, n))

    def reserve(self, n, seq=0):
        _check(lib().sa_kv_reserve(self.h, seq, n))

    def commit_accepted(self, p0, accepted, seq=0):
        """Keep verify rows [p0, p0+accepted], truncate to p0+accepted+1 and commit."""
        _check(lib().sa_kv_commit_accepted(self.h, seq, p0, accepted))

    def set_size(self, n, seq=0):
        _check(lib().sa_kv_set_size(self.h, seq, n))

    def enable_page_summaries(self, page_size=8):
        """KvStore::enable_page_summaries (kv_store.cpp:90-112): QuestLike page min / max."""
        _check(lib().sa_kv_enable_page_summaries(self.h, page_size))

    def gather(self, layer, kv_head, indices, seq=0, stream=None):
        import torch
        idx = [int(i) for i in indices]
        arr = (_i64 * max(len(idx), 1))(*idx)
        K = torch.empty((len(idx), self.d), dtype=torch.float32, device="cuda")
        V = torch.empty_like(K)
        _check(lib().sa_kv_gather(self.h, seq, layer, kv_head, arr, len(idx), K.data_ptr() if len(idx) else None,
                                  V.data_ptr() if len(idx) else None, _stream(stream)))
        return K, V

    def read(self, layer, kv_head, begin, n, seq=0, stream=None):
        import torch
        K = torch.empty((n, self.d), dtype=torch.float32, device="cuda")
        V = torch.empty_like(K)
        _check(lib().sa_kv_read(self.h, seq, layer, kv_head, begin, n, K.data_ptr() if n else None,
                                V.data_ptr() if n else None, _stream(stream)))
        return K, V


class Runner:
    """Workspaces + batch binding for the fused verify / select / draft kernels."""

    def __init__(self, cache: Cache, n_q_heads, max_rows, max_prefix, max_batch=1, sparse_ratio=0.07, k_min=16,
                 n_layers_buf=0):
        self.cache = cache
        self.Hq, self.G = n_q_heads, n_q_heads // cache.Hkv
        cfg = RunnerConfig(max_batch, n_q_heads, max_rows, max_prefix, sparse_ratio, k_min, n_layers_buf)
        h = _vp()
        _check(lib().sa_runner_create(cache.h, C.byref(cfg), C.byref(h)))
        self.h = h
        self.sparse_ratio, self.k_min = sparse_ratio, k_min

    def close(self):
        if getattr(self, "h", None):
            lib().sa_runner_destroy(self.h)
            self.h = None

    __del__ = close

    def set_batch(self, seq_ids, prefix_lens):
        n = len(seq_ids)
        s = (_i32 * n)(*seq_ids)
        p = (_i64 * n)(*prefix_lens)
        _check(lib().sa_runner_set_batch(self.h, n, s, p))
        self.B = n

    def scores(self, slot):
        ld = _i64()
        ptr = lib().sa_runner_scores(self.h, slot, C.byref(ld))
        return ptr, ld.value

    def layer_scores(self, slot):
        """Per-layer fixed-point column sums [B][ld] int64 (units of 2^-32), copied to host numpy."""
        import numpy as np
        import torch
        ld = _i64()
        ptr = lib().sa_runner_layer_scores(self.h, slot, C.byref(ld))
        torch.cuda.synchronize()
        out = np.empty(self.B * ld.value, np.int64)
        cudart_memcpy(out.ctypes.data, ptr, out.nbytes)
        return out.reshape(self.B, ld.value)

    def layer_scores_tensor(self, slot):
        """The per-layer int64 score sums of `slot` as a torch tensor ALIASING device memory ([B][ld]);
        used for the KV-head-sharded exchange (shard.exchange_layer_scores) between verify and select."""
        import torch
        ld = _i64()
        ptr = lib().sa_runner_layer_scores(self.h, slot, C.byref(ld))
        return _device_bytes(ptr, self.B * ld.value * 8).view(torch.int64).reshape(self.B, ld.value)

    def selection(self, slot, n_sets):
        """(indices [B][n_sets][k_cap] int32, counts [B][n_sets]) copied to host numpy."""
        import numpy as np
        import torch
        kc = _i32()
        ip = lib().sa_runner_indices(self.h, slot, C.byref(kc))
        cp = lib().sa_runner_counts(self.h, slot)
        torch.cuda.synchronize()
        nidx = self.B * n_sets * kc.value
        idx = np.empty(nidx, np.int32)
        cnt = np.empty(self.B * n_sets, np.int32)
        cudart_memcpy(idx.ctypes.data, ip, idx.nbytes)
        cudart_memcpy(cnt.ctypes.data, cp, cnt.nbytes)
        return idx.reshape(self.B, n_sets, kc.value), cnt.reshape(self.B, n_sets)

    def verify(self, layer, q, out, k_new=None, v_new=None, scale=None, score_row_mask=None, layer_slot=None,
               logits=None, collect_row_mask=0, score_layout=PER_LAYER, stream=None):
        R = q.shape[-2]
        if scale is None:
            scale = float((1.0 / 128 ** 0.5))
        if score_row_mask is None:
            score_row_mask = 1 | (1 << (R - 1))
        a = VerifyArgs(layer, layer if layer_slot is None else layer_slot, R, _ptr(q), _ptr(k_new), _ptr(v_new),
                       scale, score_row_mask, _ptr(out), _ptr(logits),
                       0 if logits is None else logits.shape[-1], collect_row_mask, score_layout)
        _check(lib().sa_verify_attention(self.h, C.byref(a), _stream(stream)))

    def score_weights(self, layer_slot, logits, n_rows, mode=PER_LAYER, stream=None):
        """Collect2Weights scores for layer_slot from a verify's raw logits [B][Hq][n_rows][ld]."""
        _check(lib().sa_score_weights(self.h, layer_slot, _ptr(logits), logits.shape[-1], n_rows, mode,
                                      _stream(stream)))

    def select_quest(self, layer, q, layer_slot=None, stream=None):
        """select_quest (selection.cpp:224-274) for every bound sequence; q: bf16 [B][Hq][128]."""
        _check(lib().sa_select_quest(self.h, layer, layer if layer_slot is None else layer_slot, _ptr(q),
                                     _stream(stream)))

    def select_window(self, layer_slot, sink=4, window=0, stream=None):
        """select_window (selection.cpp:209-222)."""
        _check(lib().sa_select_window(self.h, layer_slot, sink, window, _stream(stream)))

    def select(self, layer_slot, mode=PER_LAYER, rows_in_score=2, stream=None):
        a = SelectArgs(layer_slot, mode, rows_in_score)
        _check(lib().sa_select_topk(self.h, C.byref(a), _stream(stream)))

    def draft(self, layer, step, q, out, k_new=None, v_new=None, mode=PER_LAYER, scale=None, layer_slot=None,
              stream=None):
        if scale is None:
            scale = float((1.0 / 128 ** 0.5))
        a = DraftArgs(layer, layer if layer_slot is None else layer_slot, mode, step, _ptr(q), _ptr(k_new),
                      _ptr(v_new), scale, _ptr(out))
        _check(lib().sa_draft_attention(self.h, C.byref(a), _stream(stream)))

    def iteration_args(self, gamma, qv, kv_new, vv_new, qd, kd_new, vd_new, out_v, out_d, strategy=COLLECT2,
                       mode=PER_LAYER, scale=None, use_graph=True, phases=0, accepted=0):
        if scale is None:
            scale = float((1.0 / 128 ** 0.5))
        return IterationArgs(gamma, strategy, mode, scale, _ptr(qv), _ptr(kv_new), _ptr(vv_new), _ptr(qd),
                             _ptr(kd_new), _ptr(vd_new), _ptr(out_v), _ptr(out_d), int(use_graph), int(phases),
                             int(accepted))

    def iteration(self, args: IterationArgs, stream=None):
        _check(lib().sa_iteration_run(self.h, C.byref(args), _stream(stream)))

    def set_comm(self, comm: "Comm | None"):
        """Attach the KV-head group communicator (per-layer score exchange inside the iteration)."""
        self._comm = comm
        _check(lib().sa_runner_set_comm(self.h, comm.h if comm is not None else None))

    def exchange_layer_scores(self, slot, stream=None):
        _check(lib().sa_exchange_layer_scores(self.h, slot, _stream(stream)))

    def iteration_kernel_count(self, args: IterationArgs) -> int:
        return int(lib().sa_iteration_kernel_count(self.h, C.byref(args)))

    def set_dev_knob(self, name: str, value: int):
        """Dev-only tuning / tracing knob (sa_dev_set_knob); the defaults are the product settings."""
        _check(lib().sa_dev_set_knob(self.h, name.encode(), int(value)))

    def trace_dump(self, path: str) -> int:
        """Dev-only: write the verify + draft trace buffers (knob "trace") to `path`."""
        return int(lib().sa_dev_trace_dump(self.h, path.encode()))


class Comm:
    """KV-head group communicator (sa_comm): NCCL over NVLink for the per-layer score exchange.
    `unique_id` (128 bytes) comes from Comm.unique_id() on one rank of the group, shared out of band
    (e.g. torch.distributed.broadcast_object_list)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().sa_comm_unique_id(buf))
        return buf.raw

    def __init__(self, unique_id: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        h = _vp()
        _check(lib().sa_comm_create(buf, nranks, rank, C.byref(h)))
        self.h, self.nranks, self.rank = h, nranks, rank

    def info(self):
        """(nranks, rank) as NCCL reports them for this communicator."""
        n, r = _i32(), _i32()
        _check(lib().sa_comm_info(self.h, C.byref(n), C.byref(r)))
        return n.value, r.value

    def check(self):
        """Raise SpecAttnError (nccl_error) if NCCL reported an asynchronous error (comm aborted)."""
        _check(lib().sa_comm_check(self.h))

    def sync(self, stream=None, timeout_ms=-1):
        """Wait for `stream` while watching for NCCL errors / a hung peer (aborts on timeout)."""
        _check(lib().sa_comm_sync(self.h, _stream(stream), int(timeout_ms)))

    def close(self):
        if getattr(self, "h", None):
            lib().sa_comm_destroy(self.h)
            self.h = None

    __del__ = close


class QkvProjection:
    """Model-side producer: RMSNorm -> fused QKV projection -> RoPE on the device.
    w_qkv: bf16 [L][(Hq+2Hkv)*128][d_model] device tensor (rows of wq^T, wk^T, wv^T per layer),
    gain: f32 [L][d_model].  The tensors are kept referenced by the handle."""

    def __init__(self, w_qkv, gain, n_q_heads, n_kv_heads, norm_eps=1e-5, rope_theta=10000.0, rope_style=0):
        import torch
        if w_qkv.dtype != torch.bfloat16 or gain.dtype != torch.float32:
            raise SpecAttnError(1, "QkvProjection expects bf16 weights and f32 gains")
        self.w, self.gain = w_qkv.contiguous(), gain.contiguous()
        self.L, _, self.d_model = self.w.shape
        self.Hq, self.Hkv = n_q_heads, n_kv_heads
        h = _vp()
        _check(lib().sa_qkv_create(_ptr(self.w), _ptr(self.gain), self.L, self.d_model, n_q_heads, n_kv_heads,
                                   norm_eps, rope_theta, rope_style, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().sa_qkv_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_dev_knob(self, name: str, value: int):
        """Dev-only knob (sa_qkv_dev_set_knob): "trace", "dev" variant bits, "impl_tc"."""
        _check(lib().sa_qkv_dev_set_knob(self.h, name.encode(), int(value)))

    def project(self, layer, x, positions, q=None, k_new=None, v_new=None, stream=None):
        """x: f32 [B][rows][d_model] device, positions int32 [B] device -> (q, k_new, v_new) bf16."""
        import torch
        B, rows, _ = x.shape
        dev = x.device
        if q is None:
            q = torch.empty((B, self.Hq, rows, 128), dtype=torch.bfloat16, device=dev)
            k_new = torch.empty((B, rows, self.Hkv, 128), dtype=torch.bfloat16, device=dev)
            v_new = torch.empty((B, rows, self.Hkv, 128), dtype=torch.bfloat16, device=dev)
        _check(lib().sa_qkv_project(self.h, layer, _ptr(x), _ptr(positions), B, rows, _ptr(q), _ptr(k_new),
                                    _ptr(v_new), _stream(stream)))
        return q, k_new, v_new


def accept(p, draft, q=None, u=None, greedy=False, stream=None, out=None):
    """Verification acceptance on the device: p [B][g+1][V], q [B][g][V] f32,
    draft [B][g] int32, u [B][g+1] f32 -> (accepted [B], emitted [B][g+1]) int32 device tensors
    (emitted: accepted drafts, the trailing token, then -1).  out: optional preallocated pair."""
    import torch
    B, g1, V = p.shape
    if out is not None:
        acc, em = out
    else:
        acc = torch.empty((B,), dtype=torch.int32, device=p.device)
        em = torch.empty((B, g1), dtype=torch.int32, device=p.device)
    _check(lib().sa_accept(_ptr(p), _ptr(q), _ptr(draft), _ptr(u), B, g1 - 1, V, int(greedy), _ptr(acc), _ptr(em),
                           _stream(stream)))
    return acc, em


def cudart_memcpy(dst: int, src: int, nbytes: int) -> None:
    """Device->host copy of raw device memory through torch (no second CUDA runtime in Python)."""
    if nbytes == 0:
        return
    host = _device_bytes(src, nbytes).cpu().numpy()
    C.memmove(dst, host.ctypes.data, nbytes)


def _device_bytes(ptr: int, nbytes: int):
    """A uint8 CUDA tensor aliasing raw device memory (via the __cuda_array_interface__)."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}

    return torch.as_tensor(_Arr(), device="cuda")
