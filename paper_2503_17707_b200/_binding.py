"""ctypes binding of include/pipeboost.h — argument marshalling only.

Every function here has the C name it wraps and does nothing but convert Python
arguments to C types, call the library and turn a non-zero pb_status into a
PBError carrying pb_last_error(). All computation happens in libpipeboost.so;
if the library is missing the import fails loudly (there is no fallback).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpipeboost.so")

PB_MERGE_ALL = -2
PB_OK, PB_EINVAL, PB_EPARTITION, PB_EPROTOCOL, PB_ECUDA, PB_ENOMEM, PB_ENUMERIC, PB_EUNSUPPORTED = \
    0, -1, -2, -3, -4, -6, -7, -8
PB_ARCH_OPT, PB_ARCH_LLAMA = 0, 1
PB_DTYPE_BF16, PB_DTYPE_F32 = 0, 1
PB_LOAD_STAGE, PB_LOAD_INTERLEAVE = 0, 1
TARGET_BITS = {"q": 1, "k": 2, "v": 4, "o": 8, "fc1": 16, "fc2": 32, "gate": 64, "up": 128, "down": 256}


class PBError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"pb_status {status}: {msg}")
        self.status = status


class pb_model_desc(C.Structure):
    _fields_ = [("arch", C.c_int32), ("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("d_ffn", C.c_int32), ("vocab", C.c_int32), ("max_pos", C.c_int32),
                ("tied", C.c_int32), ("norm_eps", C.c_float), ("rope_theta", C.c_float), ("dtype", C.c_int32)]


class pb_adapter_desc(C.Structure):
    _fields_ = [("rank", C.c_int32), ("alpha", C.c_float), ("targets", C.c_uint32)]


class pb_plan_opts(C.Structure):
    _fields_ = [("policy", C.c_int32), ("vocab_sliced", C.c_int32), ("chunk_bytes", C.c_int64),
                ("prefill_chunks", C.c_int32), ("host_alias_layers", C.c_int32)]


class pb_plan_sizes_t(C.Structure):
    _fields_ = [("host_base_bytes", C.c_int64), ("host_adapter_bytes", C.c_int64),
                ("dev_weight_bytes", C.c_int64), ("dev_adapter_bytes", C.c_int64),
                ("n_tensors", C.c_int32), ("n_atensors", C.c_int32), ("n_chunks", C.c_int32), ("n_gpus", C.c_int32),
                ("dev_adapted_bytes", C.c_int64), ("dev_backup_bytes", C.c_int64)]


class pb_tensor_info(C.Structure):
    _fields_ = [("name", C.c_char_p), ("rows", C.c_int32), ("cols", C.c_int32), ("layer", C.c_int32),
                ("host_off", C.c_int64), ("dev_off", C.c_int64), ("bytes", C.c_int64)]


class pb_atensor_info(C.Structure):
    _fields_ = [("name", C.c_char_p), ("rows", C.c_int32), ("cols", C.c_int32), ("layer", C.c_int32),
                ("adapter", C.c_int32), ("target_bit", C.c_int32), ("is_B", C.c_int32),
                ("base_tensor", C.c_int32), ("base_row0", C.c_int32), ("off", C.c_int64), ("bytes", C.c_int64)]


class pb_rank_bufs(C.Structure):
    _fields_ = [("weights", C.c_void_p), ("weights_cap", C.c_int64), ("adapters", C.c_void_p),
                ("adapters_cap", C.c_int64), ("adapted", C.c_void_p), ("adapted_cap", C.c_int64),
                ("workspace", C.c_void_p), ("workspace_cap", C.c_int64),
                ("max_batch", C.c_int32), ("max_seq", C.c_int32), ("stream_h2d", C.c_void_p * 2),
                ("stream_merge", C.c_void_p), ("stream_nvlink", C.c_void_p), ("stream_compute", C.c_void_p),
                ("backup", C.c_void_p), ("backup_cap", C.c_int64)]


class pb_timeline_t(C.Structure):
    _fields_ = [("t_ready_ms", C.c_double), ("t_full_ms", C.c_double), ("ttft_ms", C.c_double),
                ("load_done_ms", C.c_double), ("load_bytes", C.c_int64), ("recv_bytes", C.c_int64),
                ("n_chunks", C.c_int32), ("chunk_landed_ms", C.POINTER(C.c_double)),
                ("chunk_gathered_ms", C.POINTER(C.c_double)), ("n_launches", C.c_int32),
                ("chunk_merged_ms", C.POINTER(C.c_double)), ("stage_begin_ms", C.c_double),
                ("stage_end_ms", C.c_double), ("ctx_create_ms", C.c_double)]


class pb_kernel_stat(C.Structure):
    _fields_ = [("name", C.c_char_p), ("launches", C.c_int32), ("total_ms", C.c_double), ("flops", C.c_double),
                ("bytes", C.c_double)]


class pb_kernel_event(C.Structure):
    _fields_ = [("cls", C.c_int32), ("start_ms", C.c_float), ("end_ms", C.c_float)]


_P = C.c_void_p
_SIGS = {
    "pb_plan_create": [C.POINTER(pb_model_desc), C.POINTER(pb_adapter_desc), C.c_int32, C.c_int32,
                       C.POINTER(pb_plan_opts), C.POINTER(_P)],
    "pb_plan_dump": [_P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)],
    "pb_plan_sizes": [_P, C.POINTER(pb_plan_sizes_t)],
    "pb_plan_workspace_bytes": [_P, C.c_int32, C.c_int32, C.POINTER(C.c_int64)],
    "pb_plan_tensor": [_P, C.c_int32, C.POINTER(pb_tensor_info)],
    "pb_plan_atensor": [_P, C.c_int32, C.POINTER(pb_atensor_info)],
    "pb_plan_free": [_P],
    "pb_plan_replan": [_P, _P, _P, C.POINTER(_P)],
    "pb_plan_gpu_of_rank": [_P, C.c_int32, C.POINTER(C.c_int32)],
    "pb_ctx_create": [_P, C.c_int32, _P, _P, C.POINTER(pb_rank_bufs), C.POINTER(_P)],
    "pb_ctx_export": [_P, _P, C.c_size_t, C.POINTER(C.c_size_t)],
    "pb_ctx_import_peer": [_P, C.c_int32, _P, C.c_size_t],
    "pb_ctx_link_local": [_P, C.c_int32, _P],
    "pb_trial_begin": [_P, C.c_uint32],
    "pb_load_shard": [_P],
    "pb_merge_lora": [_P, C.c_int32],
    "pb_gather_layers": [_P],
    "pb_prefill_enqueue": [_P, _P, C.c_int32, C.c_int32],
    "pb_prefill_enqueue_ex": [_P, _P, _P, C.c_int32, C.c_int32],
    "pb_prefill_wait": [_P, _P, _P],
    "pb_prefill_replay": [_P, C.c_uint32, _P, C.c_int32, C.c_int32],
    "pb_switch_adapter": [_P, C.c_int32],
    "pb_decode_step": [_P, C.c_uint32],
    "pb_ctx_set_file_source": [_P, C.c_char_p, _P, C.c_int64],
    "pb_ctx_set_replica": [_P, C.c_int32],
    "pb_epoch_create": [C.c_int32, C.c_double, C.c_int32, C.POINTER(_P)],
    "pb_epoch_set_active": [_P, C.c_int32, C.c_double],
    "pb_epoch_enqueue": [_P, C.c_int32, C.c_int64],
    "pb_epoch_next": [_P, C.c_double, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32), _P,
                      C.POINTER(C.c_int32)],
    "pb_epoch_free": [_P],
    "pb_prefill_first_token": [_P, _P, C.c_int32, C.c_int32, _P, _P],
    "pb_sync": [_P],
    "pb_timeline": [_P, C.POINTER(pb_timeline_t)],
    "pb_ctx_free": [_P],
    "pb_ctx_abort": [_P],
    "pb_ctx_set_profiling": [_P, C.c_int32],
    "pb_kernel_stats": [_P, C.POINTER(pb_kernel_stat), C.c_int32, C.POINTER(C.c_int32)],
    "pb_kernel_trace": [_P, C.POINTER(pb_kernel_event), C.c_int32, C.POINTER(C.c_int32)],
    "pb_last_error": [],
    # include/pipeboost_ops.h
    "pb_op_merge": [_P, C.c_int64, C.c_int32, C.c_int32, _P, _P, C.c_int32, C.c_float, _P],
    "pb_op_gemm": [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int32, C.c_int32, C.c_int32, _P,
                   C.c_int32, C.c_float, C.c_int32, _P, C.c_int32, _P],
    "pb_op_gemm_split": [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int32, C.c_int32, C.c_int32, _P,
                         C.c_int32, C.c_float, C.c_int32, _P, C.c_int32, C.c_int32, _P],
    "pb_op_debug_gemm": [_P, C.c_int32],
    "pb_op_merge_batch": [C.c_int32, _P, _P, _P, _P, _P, _P, C.c_int32, _P, _P],
    "pb_op_gemm_rope": [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int32, _P, C.c_int32, C.c_int32,
                        C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_float, _P, C.c_int32, _P],
    "pb_op_norm": [_P, C.c_int32, C.c_int32, _P, _P, C.c_float, _P, _P],
    "pb_op_attention": [_P, C.c_int32, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                        C.c_int32, C.c_int32, C.c_int32, C.c_float, _P],
    "pb_op_rope": [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                   C.c_int32, C.c_float, _P, _P],
    "pb_op_logits": [_P, C.c_int32, C.c_int32, _P, C.c_int32, C.c_int32, _P, C.c_int32, _P],
    "pb_op_argmax": [_P, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P],
    "pb_op_embed": [_P, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P],
}
_VOID = {"pb_plan_free", "pb_ctx_free", "pb_epoch_free"}

_lib = None


def lib():
    """Load libpipeboost.so (raises OSError if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = None if name in _VOID else (C.c_char_p if name == "pb_last_error" else C.c_int)
        _lib = L
    return _lib


def declared_symbols():
    return list(_SIGS)


def check(status):
    if status != PB_OK:
        raise PBError(status, lib().pb_last_error().decode(errors="replace"))
    return status


# --------------------------------------------------------------------------
# Thin wrappers, same names as the C ABI
# --------------------------------------------------------------------------

def model_desc(m) -> pb_model_desc:
    return pb_model_desc(PB_ARCH_OPT if m.arch == "opt" else PB_ARCH_LLAMA, m.n_layers, m.d_model, m.n_heads,
                         m.n_kv_heads, m.d_ffn, m.vocab, m.max_pos, m.tied, m.norm_eps, m.rope_theta,
                         PB_DTYPE_F32 if getattr(m, "dtype", "bf16") == "f32" else PB_DTYPE_BF16)


def adapter_desc(a) -> pb_adapter_desc:
    mask = 0
    for t in a.targets:
        mask |= TARGET_BITS[t]
    return pb_adapter_desc(a.rank, a.alpha, mask)


def plan_opts(policy="stage", vocab_sliced=0, chunk_bytes=32 << 20, prefill_chunks=1, host_alias_layers=0):
    return pb_plan_opts(PB_LOAD_STAGE if policy == "stage" else PB_LOAD_INTERLEAVE, vocab_sliced, chunk_bytes,
                        prefill_chunks, host_alias_layers)


def pb_plan_create(model, adapters, n_gpus, opts):
    md = model_desc(model)
    arr = (pb_adapter_desc * max(1, len(adapters)))(*[adapter_desc(a) for a in adapters])
    out = _P()
    check(lib().pb_plan_create(C.byref(md), arr, len(adapters), n_gpus, C.byref(opts), C.byref(out)))
    return out


def pb_plan_dump(plan) -> str:
    need = C.c_size_t(0)
    lib().pb_plan_dump(plan, None, 0, C.byref(need))
    buf = C.create_string_buffer(need.value)
    check(lib().pb_plan_dump(plan, buf, need.value, C.byref(need)))
    return buf.value.decode()


def pb_plan_sizes(plan) -> pb_plan_sizes_t:
    s = pb_plan_sizes_t()
    check(lib().pb_plan_sizes(plan, C.byref(s)))
    return s


def pb_plan_workspace_bytes(plan, batch, seq) -> int:
    v = C.c_int64(0)
    check(lib().pb_plan_workspace_bytes(plan, batch, seq, C.byref(v)))
    return v.value


def pb_plan_tensor(plan, i) -> pb_tensor_info:
    t = pb_tensor_info()
    check(lib().pb_plan_tensor(plan, i, C.byref(t)))
    return t


def pb_plan_atensor(plan, i) -> pb_atensor_info:
    t = pb_atensor_info()
    check(lib().pb_plan_atensor(plan, i, C.byref(t)))
    return t


def pb_plan_free(plan):
    lib().pb_plan_free(plan)


def pb_plan_replan(plan, alive, resident):
    """alive: sequence of 0/1 per GPU; resident: uint8 array [n_gpus, n_chunks] (1 = held)."""
    import numpy as np
    a = (C.c_int32 * len(alive))(*[int(x) for x in alive])
    r = np.ascontiguousarray(resident, dtype=np.uint8)
    out = _P()
    check(lib().pb_plan_replan(plan, a, r.ctypes.data, C.byref(out)))
    return out


def pb_plan_gpu_of_rank(plan, rank) -> int:
    v = C.c_int32(0)
    check(lib().pb_plan_gpu_of_rank(plan, rank, C.byref(v)))
    return v.value


def pb_ctx_create(plan, rank, host_base_ptr, host_adapters_ptr, bufs: pb_rank_bufs):
    out = _P()
    check(lib().pb_ctx_create(plan, rank, host_base_ptr, host_adapters_ptr, C.byref(bufs), C.byref(out)))
    return out


def pb_ctx_export(ctx) -> bytes:
    need = C.c_size_t(0)
    lib().pb_ctx_export(ctx, None, 0, C.byref(need))
    buf = C.create_string_buffer(need.value)
    check(lib().pb_ctx_export(ctx, buf, need.value, C.byref(need)))
    return buf.raw[:need.value]


def pb_ctx_import_peer(ctx, peer, blob: bytes):
    check(lib().pb_ctx_import_peer(ctx, peer, blob, len(blob)))


def pb_ctx_link_local(ctx, peer, peer_ctx):
    check(lib().pb_ctx_link_local(ctx, peer, peer_ctx))


def pb_trial_begin(ctx, epoch):
    check(lib().pb_trial_begin(ctx, epoch))


def pb_load_shard(ctx):
    check(lib().pb_load_shard(ctx))


def pb_merge_lora(ctx, adapter_id):
    check(lib().pb_merge_lora(ctx, adapter_id))


def pb_gather_layers(ctx):
    check(lib().pb_gather_layers(ctx))


def pb_prefill_enqueue(ctx, tokens_ptr, batch, seq):
    check(lib().pb_prefill_enqueue(ctx, tokens_ptr, batch, seq))


def pb_prefill_replay(ctx, epoch, tokens_ptr, batch, seq):
    check(lib().pb_prefill_replay(ctx, epoch, tokens_ptr, batch, seq))


class EpochScheduler:
    """pb_epoch_*: f2 epoch-based adapter scheduling (host side)."""

    def __init__(self, n_adapters, epoch_ms, starvation_epochs=3):
        self.h = _P()
        check(lib().pb_epoch_create(n_adapters, epoch_ms, starvation_epochs, C.byref(self.h)))

    def set_active(self, adapter, now_ms=0.0):
        check(lib().pb_epoch_set_active(self.h, adapter, now_ms))

    def enqueue(self, adapter, request_id):
        check(lib().pb_epoch_enqueue(self.h, adapter, request_id))

    def next_batch(self, now_ms, max_batch):
        import numpy as np
        a, sw, n = C.c_int32(0), C.c_int32(0), C.c_int32(0)
        ids = np.zeros(max_batch, dtype=np.int64)
        check(lib().pb_epoch_next(self.h, now_ms, max_batch, C.byref(a), C.byref(sw), ids.ctypes.data, C.byref(n)))
        if a.value == -2:
            return None, False, []
        return a.value, bool(sw.value), [int(x) for x in ids[:n.value]]

    def __del__(self):
        try:
            if self.h:
                lib().pb_epoch_free(self.h)
                self.h = None
        except Exception:
            pass


def pb_ctx_set_file_source(ctx, path, staging_ptr, staging_bytes):
    check(lib().pb_ctx_set_file_source(ctx, path.encode() if path else None, staging_ptr, staging_bytes))


def pb_decode_step(ctx, epoch):
    check(lib().pb_decode_step(ctx, epoch))


def pb_ctx_set_replica(ctx, on):
    check(lib().pb_ctx_set_replica(ctx, int(on)))


def pb_switch_adapter(ctx, adapter_id):
    check(lib().pb_switch_adapter(ctx, adapter_id))


def pb_prefill_enqueue_ex(ctx, tokens_ptr, adapter_of_seq_ptr, batch, seq):
    check(lib().pb_prefill_enqueue_ex(ctx, tokens_ptr, adapter_of_seq_ptr, batch, seq))


def pb_prefill_wait(ctx, logits_ptr, tokens_ptr):
    check(lib().pb_prefill_wait(ctx, logits_ptr, tokens_ptr))


def pb_prefill_first_token(ctx, tokens_ptr, batch, seq, logits_ptr, tokens_out_ptr):
    check(lib().pb_prefill_first_token(ctx, tokens_ptr, batch, seq, logits_ptr, tokens_out_ptr))


def pb_sync(ctx):
    check(lib().pb_sync(ctx))


def pb_timeline(ctx) -> pb_timeline_t:
    t = pb_timeline_t()
    check(lib().pb_timeline(ctx, C.byref(t)))
    return t


def pb_ctx_set_profiling(ctx, enable):
    check(lib().pb_ctx_set_profiling(ctx, 1 if enable else 0))


def pb_kernel_stats(ctx):
    n = C.c_int32(0)
    arr = (pb_kernel_stat * 16)()
    check(lib().pb_kernel_stats(ctx, arr, 16, C.byref(n)))
    return {arr[i].name.decode(): {"launches": arr[i].launches, "total_ms": arr[i].total_ms, "flops": arr[i].flops,
                                   "bytes": arr[i].bytes} for i in range(n.value)}


KCLASSES = ["merge", "gemm", "attention", "norm", "rope", "embed", "logits", "argmax", "signal"]


def pb_kernel_trace(ctx):
    n = C.c_int32(0)
    lib().pb_kernel_trace(ctx, None, 0, C.byref(n))
    arr = (pb_kernel_event * max(1, n.value))()
    check(lib().pb_kernel_trace(ctx, arr, n.value, C.byref(n)))
    return [(KCLASSES[arr[i].cls], arr[i].start_ms, arr[i].end_ms) for i in range(n.value)]


def pb_ctx_free(ctx):
    lib().pb_ctx_free(ctx)


def pb_ctx_abort(ctx):
    check(lib().pb_ctx_abort(ctx))


# --------------------------------------------------------------------------
# include/pipeboost_ops.h (device pointers as ints, stream as cudaStream_t int)
# --------------------------------------------------------------------------

def pb_op_merge(W, ldw, rows, cols, B, A, rank, scale, stream=0):
    check(lib().pb_op_merge(W, ldw, rows, cols, B, A, rank, scale, stream))


def pb_op_gemm(X, x_rows, m_begin, m_end, K, W, n_rows, N, epi, bias, relu, scale, scale_cols, out, ldo, stream=0):
    check(lib().pb_op_gemm(X, x_rows, m_begin, m_end, K, W, n_rows, N, epi, bias, relu, scale, scale_cols, out, ldo,
                           stream))


def pb_op_gemm_split(X, x_rows, m_begin, m_end, K, W, n_rows, N, epi, bias, relu, scale, scale_cols, out, ldo,
                     split_k, stream=0):
    check(lib().pb_op_gemm_split(X, x_rows, m_begin, m_end, K, W, n_rows, N, epi, bias, relu, scale, scale_cols, out,
                                 ldo, split_k, stream))


def pb_op_merge_batch(W, ldw, rows, cols, Bs, As, rank, scales, stream=0):
    """Lists of device pointers / ints / floats, one entry per job (<= 8)."""
    n = len(W)
    arr = lambda t, v: (t * n)(*v)  # noqa: E731
    check(lib().pb_op_merge_batch(n, arr(C.c_void_p, W), arr(C.c_int64, ldw), arr(C.c_int32, rows),
                                  arr(C.c_int32, cols), arr(C.c_void_p, Bs), arr(C.c_void_p, As), rank,
                                  arr(C.c_float, scales), stream))


def pb_op_debug_gemm(trace, pdl):
    check(lib().pb_op_debug_gemm(trace, pdl))


def pb_op_gemm_rope(X, x_rows, m_begin, m_end, K, W, N, out, ldo, rope_cols, hd, row0, B, T, theta, table, split_k,
                    stream):
    check(lib().pb_op_gemm_rope(X, x_rows, m_begin, m_end, K, W, N, out, ldo, rope_cols, hd, row0, B, T, theta, table,
                                split_k, stream))


def pb_op_norm(h, rows, d, gamma, beta, eps, out, stream=0):
    check(lib().pb_op_norm(h, rows, d, gamma, beta, eps, out, stream))


def pb_op_attention(qkv, ld, out, ldo, t0, t1, B, n_heads, n_kv_heads, hd, k_col0, v_col0, score_scale, stream=0):
    check(lib().pb_op_attention(qkv, ld, out, ldo, t0, t1, B, n_heads, n_kv_heads, hd, k_col0, v_col0, score_scale,
                                stream))


def pb_op_rope(qkv, ld, r0, r1, B, T, n_q, n_k, hd, k_col0, theta, table, stream=0):
    check(lib().pb_op_rope(qkv, ld, r0, r1, B, T, n_q, n_k, hd, k_col0, theta, table, stream))


def pb_op_logits(y, B, d, E, v0, v1, logits, ldl, stream=0):
    check(lib().pb_op_logits(y, B, d, E, v0, v1, logits, ldl, stream))


def pb_op_argmax(logits, B, V, ldl, tokens, nan_flag, stream=0):
    check(lib().pb_op_argmax(logits, B, V, ldl, tokens, nan_flag, stream))


def pb_op_embed(E, pos, tok, h, d, r0, r1, B, stream=0):
    check(lib().pb_op_embed(E, pos, tok, h, d, r0, r1, B, stream))
