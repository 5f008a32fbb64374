"""paper_2411_16102_b200 — thin Python binding of libblend (include/blend.h).

Blended-batch attention over a radix-tree paged KV cache: the data-parallel hot
path of BlendServe (arXiv 2411.16102).  This module only marshals arguments
(numpy host arrays -> C pointers; torch tensors -> data_ptr() and CUDA stream
handles) and calls the C ABI; every step of the path runs in libblend's
kernels.  There is no CPU fallback: if libblend.so is missing, importing the
functions raises.

    tree = build(tokens, tok_off, q_len, prompt_len, out_len, num_q_heads=32, ...)
    req_shard, shards = tree.shard(8)
    plan = tree.upload_plan(plan_buf)          # plan_buf: uint8 CUDA tensor
    attention(q, k_cache, v_cache, plan, out, lse, workspace)
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BLEND_LIB: a diagnostics build of the same sources (compile.py with BLEND_DEFINES)
LIB_PATH = os.environ.get("BLEND_LIB") or os.path.join(_HERE, "libblend.so")

OK, EINVAL, EMALFORMED, ENOSPC, ECUDA, ENOMEM, EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6
BF16, F32 = 0, 1
PATH_AUTO, PATH_GENERIC, PATH_NO_TCGEN05 = 0, 1, 2
SERIALIZE = 1
_DTYPES = {"bf16": BF16, "f32": F32}


class BlendError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status


class BuildArgs(C.Structure):
    _fields_ = [("n_req", C.c_int32), ("tok_off", C.c_void_p), ("tokens", C.c_void_p),
                ("q_len", C.c_void_p), ("prompt_len", C.c_void_p), ("out_len", C.c_void_p),
                ("global_id", C.c_void_p),
                ("num_q_heads", C.c_int32), ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("kv_dtype", C.c_int32), ("model_params", C.c_int64), ("hidden", C.c_int32),
                ("layers", C.c_int32), ("page_size", C.c_int32), ("free_pages", C.c_void_p),
                ("n_free_pages", C.c_int64), ("rows_min", C.c_int32), ("min_sep_len", C.c_int32),
                ("force_class", C.c_int32), ("split_tokens", C.c_int32), ("num_sms", C.c_int32),
                ("dense_split", C.c_int32), ("split_waste", C.c_int32)]


class TreeView(C.Structure):
    _fields_ = [("n_req", C.c_int32), ("n_nodes", C.c_int32), ("n_pages", C.c_int64)] + [
        (n, C.c_void_p) for n in (
            "node_parent", "node_start", "node_len", "node_page_off", "node_class", "node_key_cu",
            "node_key_mu", "node_first_req", "node_nreq", "page_table", "req_path_off",
            "req_path_nodes", "req_q_off", "req_class", "req_dfs_rank", "req_global_id", "req_group")]


class PlanInfo(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "n_tokens", "n_items", "n_dense_units", "n_stream_units", "n_partial_rows",
        "n_merge_tokens", "n_entries", "dense_kv_tokens", "stream_kv_tokens")]


# plan sections (csrc/internal.h order) the bench counts launches from
SEC_DENSE_UNITS, SEC_STREAM_UNITS, SEC_MERGE_TOK, SEC_DENSE_KS = 4, 5, 7, 11


class Plan(C.Structure):
    _fields_ = [("dev", C.c_void_p), ("bytes", C.c_size_t), ("off", C.c_int64 * 16),
                ("count", C.c_int64 * 16), ("num_q_heads", C.c_int32), ("num_kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("kv_dtype", C.c_int32), ("page_size", C.c_int32),
                ("dense_ctas", C.c_int32), ("n_partial_rows", C.c_int64), ("stream_entries", C.c_int64),
                ("merge_nsrc", C.c_int32), ("max_page", C.c_int32)]


class AttnArgs(C.Structure):
    _fields_ = [("q", C.c_void_p), ("k_cache", C.c_void_p), ("v_cache", C.c_void_p),
                ("n_cache_pages", C.c_int64), ("out", C.c_void_p), ("lse", C.c_void_p),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
                ("plan", C.POINTER(Plan)), ("dtype", C.c_int32), ("path", C.c_int32),
                ("flags", C.c_int32), ("events", C.c_void_p * 4)]


class SchedArgs(C.Structure):
    _fields_ = [("mem_tokens", C.c_int64), ("chunk", C.c_int32), ("step_budget", C.c_int32),
                ("policy", C.c_int32), ("max_steps", C.c_int64)]


class SchedView(C.Structure):
    _fields_ = [("n_steps", C.c_int64), ("n_entries", C.c_int64), ("n_req", C.c_int32),
                ("n_admitted", C.c_int32)] + [(n, C.c_void_p) for n in (
                    "step_off", "req", "n_cached", "q", "order", "side", "m_left")] + [
                ("cached_prompt_tokens", C.c_int64), ("optimal_cached_tokens", C.c_int64)]


SCHED_DUAL, SCHED_DFS = 0, 1

_lib = None

EXPORTS = {
    "blend_last_error": (C.c_char_p, []),
    "blend_abi_version": (C.c_int, []),
    "blend_tree_build": (C.c_int, [C.POINTER(BuildArgs), C.POINTER(C.c_void_p)]),
    "blend_tree_get_view": (C.c_int, [C.c_void_p, C.POINTER(TreeView)]),
    "blend_tree_free": (None, [C.c_void_p]),
    "blend_tree_dump": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "blend_shard": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_void_p]),
    "blend_plan_get_info": (C.c_int, [C.c_void_p, C.POINTER(PlanInfo)]),
    "blend_plan_bytes": (C.c_size_t, [C.c_void_p]),
    "blend_workspace_bytes": (C.c_size_t, [C.c_void_p]),
    "blend_plan_upload": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.POINTER(Plan)]),
    "blend_attention": (C.c_int, [C.POINTER(AttnArgs), C.c_void_p]),
    "blend_fill_kv": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_uint64, C.c_void_p]),
    "blend_fill_q": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                               C.c_int64, C.c_uint64, C.c_float, C.c_void_p]),
    "blend_l2_flush": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p]),
    "blend_schedule_build": (C.c_int, [C.c_void_p, C.POINTER(SchedArgs), C.POINTER(C.c_void_p)]),
    "blend_schedule_get_view": (C.c_int, [C.c_void_p, C.POINTER(SchedView)]),
    "blend_schedule_free": (None, [C.c_void_p]),
}


def lib():
    """Load libblend.so (built in-tree by paper_2411_16102_b200.compile); raise if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libblend.so not built ({LIB_PATH}); run "
                              "`python -m paper_2411_16102_b200.compile` — there is no fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int):
    if status != OK:
        raise BlendError(status, lib().blend_last_error().decode(errors="replace"))


def _arr(x, dtype):
    a = np.ascontiguousarray(np.asarray(x, dtype=dtype))
    return a, a.ctypes.data


def _stream_handle(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


class Tree:
    """Host-owned descriptor tree (blend_tree*)."""

    def __init__(self, handle: int, keep=None):
        self._h = C.c_void_p(handle)
        self._keep = keep

    @property
    def handle(self):
        return self._h

    def free(self):
        if self._h and self._h.value:
            lib().blend_tree_free(self._h)
            self._h = C.c_void_p(None)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def view(self) -> dict:
        v = TreeView()
        _check(lib().blend_tree_get_view(self._h, C.byref(v)))
        R, N, P = v.n_req, v.n_nodes, v.n_pages
        total_path = int(np.ctypeslib.as_array(C.cast(v.req_path_off, C.POINTER(C.c_int64)), (R + 1,))[-1])

        def get(ptr, ctype, n, dt):
            if n == 0:
                return np.zeros(0, dtype=dt)
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), (n,)).astype(dt, copy=True)
        return dict(
            n_req=R, n_nodes=N, n_pages=P,
            node_parent=get(v.node_parent, C.c_int32, N, np.int32),
            node_start=get(v.node_start, C.c_int32, N, np.int32),
            node_len=get(v.node_len, C.c_int32, N, np.int32),
            node_page_off=get(v.node_page_off, C.c_int64, N + 1, np.int64),
            node_class=get(v.node_class, C.c_uint8, N, np.uint8),
            node_key_cu=get(v.node_key_cu, C.c_uint64, 2 * N, np.uint64).reshape(N, 2),
            node_key_mu=get(v.node_key_mu, C.c_uint64, 2 * N, np.uint64).reshape(N, 2),
            node_first_req=get(v.node_first_req, C.c_int32, N, np.int32),
            node_nreq=get(v.node_nreq, C.c_int32, N, np.int32),
            page_table=get(v.page_table, C.c_int32, P, np.int32),
            req_path_off=get(v.req_path_off, C.c_int64, R + 1, np.int64),
            req_path_nodes=get(v.req_path_nodes, C.c_int32, total_path, np.int32),
            req_q_off=get(v.req_q_off, C.c_int64, R + 1, np.int64),
            req_class=get(v.req_class, C.c_uint8, R, np.uint8),
            req_dfs_rank=get(v.req_dfs_rank, C.c_int32, R, np.int32),
            req_global_id=get(v.req_global_id, C.c_int64, R, np.int64),
            req_group=get(v.req_group, C.c_int32, R, np.int32),
        )

    def dump(self) -> str:
        need = C.c_size_t(0)
        lib().blend_tree_dump(self._h, None, 0, C.byref(need))
        buf = C.create_string_buffer(need.value)
        _check(lib().blend_tree_dump(self._h, buf, need.value, C.byref(need)))
        return buf.value.decode()

    def plan_info(self) -> dict:
        i = PlanInfo()
        _check(lib().blend_plan_get_info(self._h, C.byref(i)))
        return {n: getattr(i, n) for n, _ in PlanInfo._fields_}

    @property
    def plan_bytes(self) -> int:
        return int(lib().blend_plan_bytes(self._h))

    @property
    def workspace_bytes(self) -> int:
        return int(lib().blend_workspace_bytes(self._h))

    def shard(self, n_shards: int, kappa: int = 213,
              shard_free_pages: Optional[Sequence[Optional[np.ndarray]]] = None
              ) -> Tuple[np.ndarray, List[Optional["Tree"]]]:
        R = self.view_n_req()
        req_shard = np.zeros(R, dtype=np.int32)
        handles = (C.c_void_p * n_shards)()
        fp_ptrs = fp_n = keep = None
        if shard_free_pages is not None:
            keep = [None if x is None else np.ascontiguousarray(x, dtype=np.int32) for x in shard_free_pages]
            fp_ptrs = (C.c_void_p * n_shards)(*[None if x is None else x.ctypes.data for x in keep])
            fp_n = (C.c_int64 * n_shards)(*[0 if x is None else len(x) for x in keep])
        _check(lib().blend_shard(self._h, n_shards, kappa,
                                 C.cast(fp_ptrs, C.c_void_p) if fp_ptrs is not None else None,
                                 C.cast(fp_n, C.c_void_p) if fp_n is not None else None,
                                 req_shard.ctypes.data, C.cast(handles, C.c_void_p)))
        return req_shard, [Tree(h) if h else None for h in handles]

    def view_n_req(self) -> int:
        v = TreeView()
        _check(lib().blend_tree_get_view(self._h, C.byref(v)))
        return v.n_req

    def schedule(self, mem_tokens: int, chunk: int = 512, step_budget: int = 8192, policy: int = 0,
                 max_steps: int = 0) -> dict:
        """blend_schedule_build on this (whole-workload) tree: the dual-scanner batch stream."""
        a = SchedArgs(mem_tokens, chunk, step_budget, policy, max_steps)
        h = C.c_void_p()
        _check(lib().blend_schedule_build(self._h, C.byref(a), C.byref(h)))
        try:
            v = SchedView()
            _check(lib().blend_schedule_get_view(h, C.byref(v)))

            def get(ptr, ctype, n, dt):
                if n == 0:
                    return np.zeros(0, dtype=dt)
                return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), (n,)).astype(dt, copy=True)
            E, S = v.n_entries, v.n_steps
            return dict(n_steps=S, step_off=get(v.step_off, C.c_int64, S + 1, np.int64),
                        req=get(v.req, C.c_int32, E, np.int32), n_cached=get(v.n_cached, C.c_int32, E, np.int32),
                        q=get(v.q, C.c_int32, E, np.int32), order=get(v.order, C.c_int32, v.n_admitted, np.int32),
                        side=get(v.side, C.c_uint8, v.n_req, np.uint8), m_left=get(v.m_left, C.c_int64, S, np.int64),
                        cached_prompt_tokens=v.cached_prompt_tokens, optimal_cached_tokens=v.optimal_cached_tokens)
        finally:
            lib().blend_schedule_free(h)

    def upload_plan(self, dev_buf, stream=None) -> Plan:
        """Copy the plan into dev_buf (a CUDA tensor of >= plan_bytes bytes)."""
        plan = Plan()
        nbytes = dev_buf.numel() * dev_buf.element_size()
        _check(lib().blend_plan_upload(self._h, C.c_void_p(dev_buf.data_ptr()), nbytes,
                                       C.c_void_p(_stream_handle(stream)), C.byref(plan)))
        plan._buf = dev_buf
        return plan


def build(tokens, tok_off, q_len, prompt_len, out_len, *, num_q_heads, num_kv_heads, head_dim,
          kv_dtype="bf16", model_params=8_030_261_248, hidden=4096, layers=32, page_size=64,
          free_pages=None, global_id=None, rows_min=128, min_sep_len=128, force_class=0,
          split_tokens=0, num_sms=148, dense_split=0, split_waste=0) -> Tree:
    """blend_tree_build on host arrays (numpy-convertible).  Array lengths are checked
    here (the C side trusts n_req = len(q_len)): ValueError on a mismatch."""
    keep = []
    R = len(q_len)
    for name, arr, n in (("tok_off", tok_off, R + 1), ("prompt_len", prompt_len, R), ("out_len", out_len, R)) + \
            ((("global_id", global_id, R),) if global_id is not None else ()):
        if len(arr) != n:
            raise ValueError(f"{name} has {len(arr)} entries, expected {n} (n_req = len(q_len) = {R})")
    if R and (int(tok_off[0]) != 0 or int(tok_off[-1]) != len(tokens)):
        raise ValueError(f"tok_off must run from 0 to len(tokens) = {len(tokens)}")
    tok_off, p_off = _arr(tok_off, np.int64); keep.append(tok_off)
    tokens, p_tok = _arr(tokens, np.int32); keep.append(tokens)
    q_len, p_q = _arr(q_len, np.int32); keep.append(q_len)
    prompt_len, p_p = _arr(prompt_len, np.int32); keep.append(prompt_len)
    out_len, p_d = _arr(out_len, np.int32); keep.append(out_len)
    a = BuildArgs()
    a.n_req = len(q_len)
    a.tok_off, a.tokens, a.q_len, a.prompt_len, a.out_len = p_off, p_tok, p_q, p_p, p_d
    if global_id is not None:
        gid, a.global_id = _arr(global_id, np.int64); keep.append(gid)
    a.num_q_heads, a.num_kv_heads, a.head_dim = num_q_heads, num_kv_heads, head_dim
    a.kv_dtype = _DTYPES[kv_dtype] if isinstance(kv_dtype, str) else int(kv_dtype)
    a.model_params, a.hidden, a.layers, a.page_size = model_params, hidden, layers, page_size
    if free_pages is not None:
        fp, a.free_pages = _arr(free_pages, np.int32); keep.append(fp)
        a.n_free_pages = len(fp)
    a.rows_min, a.min_sep_len, a.force_class = rows_min, min_sep_len, force_class
    a.split_tokens, a.num_sms, a.dense_split = split_tokens, num_sms, dense_split
    a.split_waste = split_waste
    h = C.c_void_p()
    _check(lib().blend_tree_build(C.byref(a), C.byref(h)))
    return Tree(h.value)


def _torch_dtype_code(t) -> int:
    name = str(t.dtype)
    if name == "torch.bfloat16":
        return BF16
    if name == "torch.float32":
        return F32
    return -1                      # rejected by blend_attention (EINVAL)


def attention(q, k_cache, v_cache, plan: Plan, out, lse, workspace, *, n_cache_pages: int,
              stream=None, path: int = PATH_AUTO, events=None, flags: int = 0) -> None:
    """blend_attention: enqueue on `stream` (default: torch's current stream)."""
    a = AttnArgs()
    a.q, a.k_cache, a.v_cache = q.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr()
    a.n_cache_pages = int(n_cache_pages)
    a.out, a.lse = out.data_ptr(), lse.data_ptr()
    if workspace is not None:
        a.workspace = workspace.data_ptr()
        a.workspace_bytes = workspace.numel() * workspace.element_size()
    a.plan = C.pointer(plan)
    a.dtype = _torch_dtype_code(q)
    a.path = path
    a.flags = flags
    if events:
        for i, ev in enumerate(events[:4]):
            a.events[i] = None if ev is None else ev.cuda_event
    _check(lib().blend_attention(C.byref(a), C.c_void_p(_stream_handle(stream))))


def fill_kv(k_cache, v_cache, kv_dtype, num_kv_heads, head_dim, page_size, page_ids, page_count,
            page_hash, seed, stream=None, kv_head0=0):
    """blend_fill_kv (device arrays page_ids/page_count/page_hash as torch tensors)."""
    _check(lib().blend_fill_kv(k_cache.data_ptr(), v_cache.data_ptr(), _DTYPES.get(kv_dtype, kv_dtype),
                               num_kv_heads, kv_head0, head_dim, page_size, page_ids.data_ptr(),
                               page_count.data_ptr(), page_hash.data_ptr(), page_ids.numel(),
                               C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), C.c_void_p(_stream_handle(stream))))


def fill_q(q, dtype, num_q_heads, head_dim, row_gid, row_t, seed, scale_q=1.0, stream=None, head0=0):
    _check(lib().blend_fill_q(q.data_ptr(), _DTYPES.get(dtype, dtype), num_q_heads, head0, head_dim,
                              row_gid.data_ptr(), row_t.data_ptr(), row_gid.numel(),
                              C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), C.c_float(scale_q),
                              C.c_void_p(_stream_handle(stream))))


def set_stats(buf=None):
    """Diagnostics only: point the calling thread's subsequent blend_attention calls at a
    device uint64[8] buffer of softmax path counters (csrc/common.cuh STAT_*), or detach
    (None).  Production calls leave it detached."""
    L = lib()
    f = L.blend_internal_set_stats
    f.restype, f.argtypes = C.c_int, [C.c_void_p]
    f(None if buf is None else C.c_void_p(buf.data_ptr()))


STAT_NAMES = ["dense_blocks", "dense_slow", "dense_slow_late", "dense_rescale", "stream_stages",
              "stream_rescale", "tail_zeroed"]


def l2_flush(buf, stream=None):
    _check(lib().blend_l2_flush(buf.data_ptr(), buf.numel() * buf.element_size(),
                                C.c_void_p(_stream_handle(stream))))
