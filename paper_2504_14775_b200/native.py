"""ctypes binding of the C-ABI in include/gllm.h (libgllm.so, built in-tree for sm_100a).

There is no fallback: if the library is missing or a call fails, this module
raises (`NativeError` carries `gllm_last_error()`). Device buffers are passed
as raw pointers taken from torch tensors; streams as `cudaStream_t` handles.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import NativeError

# GLLM_LIB: A/B comparisons against another build (tools only); the default is the in-tree library
LIB_PATH = os.environ.get("GLLM_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgllm.so")

SEQ_FIELDS = 5

# Every symbol include/gllm.h declares (checked by tests/test_native_abi.py).
EXPORTS = (
    "gllm_version", "gllm_last_error", "gllm_attention_q_tile", "gllm_stage_workspace_bytes",
    "gllm_stage_forward", "gllm_commit_tokens", "gllm_gemm_workspace_reset", "gllm_gemm_bf16", "gllm_gemm_swiglu_bf16", "gllm_gemm_qkv_rope_bf16",
    "gllm_rmsnorm", "gllm_silu_mul",
    "gllm_prepare_batch", "gllm_embed", "gllm_rope_kv_write", "gllm_attn_mixed_paged", "gllm_attn_mixed_paged_split", "gllm_attn_mixed_paged_auto",
    "gllm_attn_split_workspace_bytes", "gllm_argmax",
    "gllm_launch_count", "gllm_profile_begin", "gllm_profile_end", "gllm_meta_errors",
)

META_ERRORS = {1: "block-table delta out of range", 2: "prompt header out of range",
               4: "sequence row / position out of range", 8: "token position maps to an invalid page"}


class Dims(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("d_model", C.c_int), ("n_heads", C.c_int), ("n_kv_heads", C.c_int),
                ("head_dim", C.c_int), ("d_ff", C.c_int), ("vocab", C.c_int), ("qkv_bias", C.c_int),
                ("rms_eps", C.c_float), ("page_size", C.c_int), ("num_pages", C.c_int), ("max_rows", C.c_int),
                ("max_pages_per_row", C.c_int), ("max_seq_len", C.c_int), ("max_tokens", C.c_int),
                ("max_emit", C.c_int), ("fused_norm", C.c_int)]


class Layer(C.Structure):
    _fields_ = [("attn_norm", C.c_void_p), ("w_qkv", C.c_void_p), ("b_qkv", C.c_void_p), ("w_o", C.c_void_p),
                ("mlp_norm", C.c_void_p), ("w_gate_up", C.c_void_p), ("w_down", C.c_void_p)]


class Stage(C.Structure):
    _fields_ = [("dims", Dims), ("is_first", C.c_int), ("is_last", C.c_int), ("embed", C.c_void_p),
                ("final_norm", C.c_void_p), ("lm_head", C.c_void_p), ("layers", C.POINTER(Layer)),
                ("k_cache", C.c_void_p), ("v_cache", C.c_void_p), ("block_table", C.c_void_p),
                ("token_hist", C.c_void_p), ("rope", C.c_void_p), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t)]


class Batch(C.Structure):
    _fields_ = [("n_seqs", C.c_int), ("n_tokens", C.c_int), ("n_emit", C.c_int), ("n_work", C.c_int),
                ("n_prefill_work", C.c_int), ("n_deltas", C.c_int), ("n_prompts", C.c_int), ("meta", C.c_void_p), ("hidden", C.c_void_p),
                ("sampled", C.c_void_p), ("logits", C.c_void_p), ("host_seq_info", C.c_void_p)]


class ProfileEntry(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int), ("total_ms", C.c_double),
                ("flops", C.c_double), ("bytes", C.c_double)]


_lib = None


def load() -> C.CDLL:
    """Load libgllm.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeError("load", -1, f"{LIB_PATH} missing: run `python -m paper_2504_14775_b200.build`")
    lib = C.CDLL(LIB_PATH)
    vp, i, sz, f = C.c_void_p, C.c_int, C.c_size_t, C.c_float
    sig = {
        "gllm_version": (i, []),
        "gllm_last_error": (C.c_char_p, []),
        "gllm_attention_q_tile": (i, [i, i]),
        "gllm_stage_workspace_bytes": (sz, [C.POINTER(Dims)]),
        "gllm_stage_forward": (i, [C.POINTER(Stage), C.POINTER(Batch), vp]),
        "gllm_commit_tokens": (i, [C.POINTER(Stage), C.POINTER(Batch), vp, vp]),
        "gllm_gemm_workspace_reset": (i, [vp, vp]),
        "gllm_gemm_bf16": (i, [vp, i, vp, i, vp, i, i, i, i, vp, vp, i, i, i, vp, sz, vp]),
        "gllm_gemm_swiglu_bf16": (i, [vp, i, vp, i, vp, i, i, i, i, i, i, vp, sz, vp]),
        "gllm_gemm_qkv_rope_bf16": (i, [vp, i, vp, i, vp, vp, i, i, i, i, vp, vp, vp, vp, vp, i, i, i, vp, sz, vp]),
        "gllm_rmsnorm": (i, [vp, i, vp, vp, vp, i, i, f, vp]),
        "gllm_silu_mul": (i, [vp, i, vp, i, vp]),
        "gllm_prepare_batch": (i, [C.POINTER(Stage), C.POINTER(Batch), vp, vp, vp, vp, vp]),
        "gllm_embed": (i, [vp, i, vp, i, vp, vp]),
        "gllm_rope_kv_write": (i, [vp, i, i, i, i, vp, vp, vp, vp, vp, i, vp]),
        "gllm_attn_mixed_paged": (i, [vp, vp, vp, i, i, vp, i, i, vp, vp, i, i, i, i, vp, vp]),
        "gllm_attn_mixed_paged_split": (i, [vp, vp, vp, i, i, vp, i, i, vp, vp, i, i, i, i, vp, i, vp, C.c_size_t,
                                            vp]),
        "gllm_attn_mixed_paged_auto": (i, [vp, vp, vp, i, i, vp, i, i, vp, vp, i, i, i, i, vp, vp, vp, vp,
                                           C.c_size_t, vp]),
        "gllm_attn_split_workspace_bytes": (C.c_size_t, [i, i, i]),
        "gllm_argmax": (i, [vp, i, i, vp, vp]),
        "gllm_launch_count": (C.c_ulonglong, []),
        "gllm_profile_begin": (i, []),
        "gllm_profile_end": (i, [C.POINTER(ProfileEntry), i, C.POINTER(i)]),
        "gllm_meta_errors": (C.c_uint32, [i]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def call(name: str, *args) -> None:
    """Invoke a gllm_* entry point; raise NativeError on a non-zero return."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        raise NativeError(name, rc, lib.gllm_last_error().decode(errors="replace"))


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


_profiling = False


def profile_begin() -> None:
    global _profiling
    call("gllm_profile_begin")
    _profiling = True


def profiling() -> bool:
    """The native per-launch profiler is on (its CUDA events cannot live inside a captured graph)."""
    return _profiling


def profile_end() -> dict[str, dict]:
    """Aggregated per-kernel-class CUDA-event timings captured since `profile_begin`."""
    global _profiling
    arr = (ProfileEntry * 64)()
    n = C.c_int(0)
    call("gllm_profile_end", arr, 64, C.byref(n))
    _profiling = False
    return {arr[i].name.decode(): {"launches": arr[i].launches, "total_ms": arr[i].total_ms,
                                   "flops": arr[i].flops, "bytes": arr[i].bytes} for i in range(n.value)}


def check_meta_errors() -> None:
    """Raise if any micro-batch's metadata failed the device bounds checks (gllm_meta_errors)."""
    v = int(load().gllm_meta_errors(1))
    if v:
        why = ", ".join(m for b, m in META_ERRORS.items() if v & b)
        raise NativeError("gllm_meta_errors", v, f"device metadata bounds check failed: {why}")


def launch_count() -> int:
    return int(load().gllm_launch_count())
