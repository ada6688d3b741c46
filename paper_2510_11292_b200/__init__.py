"""Python binding of the LouisKV B200 C ABI (include/louiskv.h).

Argument marshalling only: every computation runs in the CUDA kernels of
``liblouiskv.so`` (built in-tree for sm_100a by ``build.py``). There is no CPU
fallback — importing this package without the built library raises.

Functions keep the C names without the ``louiskv_`` prefix and take torch
tensors (device memory / streams come from PyTorch: plumbing only).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LOUISKV_LIB", os.path.join(HERE, "liblouiskv.so"))  # (override: profiling build)

OK, ERR_INVALID_ARG, ERR_STATE, ERR_CAPACITY, ERR_OOM_DEVICE, ERR_OOM_HOST, ERR_CUDA, ERR_NOT_IMPLEMENTED = range(8)
TRIG_PREV_STEP, TRIG_LAST_RETRIEVAL = 0, 1
BOUNDARY_PER_LAYER, BOUNDARY_SHARED = 0, 1
KMEANS_TC, KMEANS_SIMT = 0, 1
UNITS_KMEANS, UNITS_PAGES = 0, 1
FETCH_ZERO_COPY, FETCH_BATCHED_DMA = 0, 1
POOL_BF16, POOL_FP8_E4M3 = 0, 1

_STATUS = {0: "OK", 1: "INVALID_ARG", 2: "STATE", 3: "CAPACITY", 4: "OOM_DEVICE", 5: "OOM_HOST", 6: "CUDA",
           7: "NOT_IMPLEMENTED"}

# ABI symbols declared in include/louiskv.h (checked by tests/test_abi.py)
SYMBOLS = ["louiskv_create", "louiskv_destroy", "louiskv_cluster_prompt", "louiskv_prompt_fence", "louiskv_set_prompt_units",
           "louiskv_should_retrieve", "louiskv_retrieve", "louiskv_append_output", "louiskv_sparse_attn",
           "louiskv_append_attn", "louiskv_decode_layer",
           "louiskv_get_selection", "louiskv_get_units", "louiskv_get_unit_positions", "louiskv_get_working_set",
           "louiskv_get_stats", "louiskv_get_memory", "louiskv_set_prefill_timing", "louiskv_get_prefill_times",
           "louiskv_state_save", "louiskv_state_restore", "louiskv_get_pool_numa_node", "louiskv_last_error",
           "louiskv_version"]


class LouisKVError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"louiskv {_STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("kv_head_begin", ctypes.c_int32), ("kv_head_count", ctypes.c_int32),
                ("max_batch", ctypes.c_int32), ("max_prompt_len", ctypes.c_int64), ("max_output_len", ctypes.c_int64),
                ("budget_tokens", ctypes.c_int32), ("sink_tokens", ctypes.c_int32), ("window_tokens", ctypes.c_int32),
                ("tau", ctypes.c_double), ("avg_cluster_size", ctypes.c_int32), ("kmeans_iters", ctypes.c_int32),
                ("kmeans_impl", ctypes.c_int32), ("full_cache_layers", ctypes.c_uint64),
                ("trigger_ref", ctypes.c_int32), ("boundary_mode", ctypes.c_int32), ("shared_layer", ctypes.c_int32),
                ("max_open_segment", ctypes.c_int32), ("fetch_mode", ctypes.c_int32), ("device", ctypes.c_int32),
                ("attn_impl", ctypes.c_int32), ("trigger_stride", ctypes.c_int32), ("prompt_units", ctypes.c_int32),
                ("index_offload", ctypes.c_int32), ("pool_dtype", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ("retrievals", "units_scored", "units_selected", "units_reused",
                                                "units_fetched", "bytes_h2d", "bytes_d2h", "segments_evicted",
                                                "kmeans_tc_iters", "kmeans_simt_iters", "dma_copies")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class PrefillTimes(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("init_ms", "assign_ms", "sort_ms", "update_ms", "stage_ms", "d2h_ms")] + \
               [(n, ctypes.c_uint64) for n in ("assign_flops", "keys", "d2h_bytes", "assign_passes")] + \
               [("calls", ctypes.c_int32)]

    def as_dict(self):
        return {n: (float(getattr(self, n)) if t is ctypes.c_double else int(getattr(self, n)))
                for n, t in self._fields_}


_lib = None


def lib():
    """Load liblouiskv.so (in-tree). Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, u8p = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
        L.louiskv_create.argtypes = [ctypes.POINTER(Config), ctypes.POINTER(ctypes.c_void_p)]
        L.louiskv_destroy.argtypes = [vp]
        L.louiskv_destroy.restype = None
        L.louiskv_cluster_prompt.argtypes = [vp, i32, vp, vp, i64, i64, i64, i32, i64, vp]
        L.louiskv_prompt_fence.argtypes = [vp, vp]
        L.louiskv_set_prompt_units.argtypes = [vp, i32, vp, vp, i64, i64, i64, i32, i64, i32, vp, vp, vp]
        L.louiskv_should_retrieve.argtypes = [vp, i32, vp, i64, u8p, vp, vp]
        L.louiskv_retrieve.argtypes = [vp, i32, vp, i64, vp]
        L.louiskv_append_output.argtypes = [vp, i32, vp, vp, i64, vp]
        L.louiskv_sparse_attn.argtypes = [vp, i32, vp, i64, vp, vp, vp]
        L.louiskv_append_attn.argtypes = [vp, i32, vp, vp, i64, vp, i64, vp, vp, vp]
        L.louiskv_decode_layer.argtypes = [vp, i32, vp, i64, vp, vp, i64, vp, vp, vp, vp, vp]
        L.louiskv_get_selection.argtypes = [vp, i32, i32, i32, vp, i32, ctypes.POINTER(ctypes.c_int32)]
        L.louiskv_get_units.argtypes = [vp, i32, i32, i32, i32, vp, vp, vp, ctypes.POINTER(ctypes.c_int32)]
        L.louiskv_get_unit_positions.argtypes = [vp, i32, i32, i32, vp, i64, ctypes.POINTER(ctypes.c_int64)]
        L.louiskv_get_working_set.argtypes = [vp, i32, i32, i32, vp, vp, i32, ctypes.POINTER(ctypes.c_int32)]
        L.louiskv_get_stats.argtypes = [vp, ctypes.POINTER(Stats)]
        L.louiskv_get_memory.argtypes = [vp, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
        L.louiskv_set_prefill_timing.argtypes = [vp, i32]
        L.louiskv_get_prefill_times.argtypes = [vp, ctypes.POINTER(PrefillTimes)]
        L.louiskv_state_save.argtypes = [vp, vp]
        L.louiskv_state_restore.argtypes = [vp, vp]
        L.louiskv_get_pool_numa_node.argtypes = [vp, ctypes.POINTER(ctypes.c_int32)]
        L.louiskv_last_error.argtypes = [vp]
        L.louiskv_last_error.restype = ctypes.c_char_p
        L.louiskv_version.restype = ctypes.c_char_p
        for name in SYMBOLS:
            f = getattr(L, name)
            if f.restype is None and name not in ("louiskv_destroy",):
                f.restype = ctypes.c_int
            elif name not in ("louiskv_destroy", "louiskv_last_error", "louiskv_version"):
                f.restype = ctypes.c_int
        _lib = L
    return _lib


def version() -> str:
    return lib().louiskv_version().decode()


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    return int(t.data_ptr())


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return int(torch.cuda.current_stream().cuda_stream)
    return int(getattr(stream, "cuda_stream", stream))


def make_config(cfg, kv_head_begin=0, kv_head_count=None, max_batch=None, trigger_ref=TRIG_PREV_STEP,
                boundary_mode=BOUNDARY_PER_LAYER, shared_layer=0, max_open_segment=0, kmeans_impl=KMEANS_TC,
                device=0, max_output_len=None, attn_impl=0, trigger_stride=0, prompt_units=0,
                fetch_mode=FETCH_ZERO_COPY, index_offload=0, pool_dtype=0) -> Config:
    """Build the C config from a synth.configs.Config-like object (plain numbers)."""
    mask = 0
    for l in cfg.full_cache_layers:
        mask |= 1 << l
    return Config(num_layers=cfg.num_layers, num_q_heads=cfg.num_q_heads, num_kv_heads=cfg.num_kv_heads,
                  head_dim=cfg.head_dim, kv_head_begin=kv_head_begin,
                  kv_head_count=cfg.num_kv_heads - kv_head_begin if kv_head_count is None else kv_head_count,
                  max_batch=cfg.batch if max_batch is None else max_batch, max_prompt_len=cfg.prompt_len,
                  max_output_len=cfg.max_output_len if max_output_len is None else max_output_len,
                  budget_tokens=cfg.budget_tokens, sink_tokens=cfg.sink_tokens, window_tokens=cfg.window_tokens,
                  tau=cfg.tau, avg_cluster_size=cfg.avg_cluster_size, kmeans_iters=cfg.kmeans_iters,
                  kmeans_impl=kmeans_impl, full_cache_layers=mask, trigger_ref=trigger_ref,
                  boundary_mode=boundary_mode, shared_layer=shared_layer, max_open_segment=max_open_segment,
                  fetch_mode=fetch_mode, device=device, attn_impl=attn_impl, trigger_stride=trigger_stride,
                  prompt_units=prompt_units, index_offload=index_offload, pool_dtype=pool_dtype)


class Context:
    """Owning wrapper of a louiskv_ctx*. Methods mirror the C ABI one to one."""

    def __init__(self, config: Config):
        self._L = lib()
        self.cfg = config
        h = ctypes.c_void_p()
        s = self._L.louiskv_create(ctypes.byref(config), ctypes.byref(h))
        if s != OK:
            raise LouisKVError(s, "louiskv_create failed")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self._L.louiskv_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, s):
        if s != OK:
            raise LouisKVError(s, self._L.louiskv_last_error(self.h).decode())

    # --- ABI calls ---------------------------------------------------------
    def cluster_prompt(self, layer, k, v, stream=None):
        """k, v: bf16 [b, P, Hkv_owned, d] (any strides with d contiguous)."""
        b, P = k.shape[0], k.shape[1]
        self._chk(self._L.louiskv_cluster_prompt(self.h, layer, _ptr(k), _ptr(v), k.stride(0), k.stride(1),
                                                 k.stride(2), b, P, _stream(stream)))

    def prompt_fence(self, stream=None):
        """Make `stream` wait for every pending prompt offload (copy-engine D2H into the pool)."""
        self._chk(self._L.louiskv_prompt_fence(self.h, _stream(stream)))

    def set_prompt_units(self, layer, k, v, assign: np.ndarray, centroids: np.ndarray, stream=None):
        b, P = k.shape[0], k.shape[1]
        assign = np.ascontiguousarray(assign, dtype=np.int32)
        centroids = np.ascontiguousarray(centroids, dtype=np.float32)
        n_clusters = centroids.shape[-2] if centroids.ndim >= 2 else 0
        self._chk(self._L.louiskv_set_prompt_units(self.h, layer, _ptr(k), _ptr(v), k.stride(0), k.stride(1),
                                                   k.stride(2), b, P, n_clusters, assign.ctypes.data,
                                                   centroids.ctypes.data, _stream(stream)))

    def should_retrieve(self, layer, q_all, flag_out=None, r_out=None, stream=None):
        self._chk(self._L.louiskv_should_retrieve(self.h, layer, _ptr(q_all), q_all.stride(0), _ptr(flag_out),
                                                  _ptr(r_out), _stream(stream)))

    def retrieve(self, layer, q_own, stream=None):
        self._chk(self._L.louiskv_retrieve(self.h, layer, _ptr(q_own), q_own.stride(0), _stream(stream)))

    def append_output(self, layer, k_t, v_t, stream=None):
        assert k_t.stride(0) == v_t.stride(0)
        self._chk(self._L.louiskv_append_output(self.h, layer, _ptr(k_t), _ptr(v_t), k_t.stride(0), _stream(stream)))

    def sparse_attn(self, layer, q_own, out, out_f32=None, stream=None):
        self._chk(self._L.louiskv_sparse_attn(self.h, layer, _ptr(q_own), q_own.stride(0), _ptr(out), _ptr(out_f32),
                                              _stream(stream)))

    def append_attn(self, layer, k_t, v_t, q_own, out, out_f32=None, stream=None):
        """Fused append_output + sparse_attn (one clustered launch on retrieval layers)."""
        assert k_t.stride(0) == v_t.stride(0)
        self._chk(self._L.louiskv_append_attn(self.h, layer, _ptr(k_t), _ptr(v_t), k_t.stride(0), _ptr(q_own),
                                              q_own.stride(0), _ptr(out), _ptr(out_f32), _stream(stream)))

    def decode_layer(self, layer, q_all, k_t, v_t, out, out_f32=None, flag_out=None, r_out=None, stream=None):
        """One whole decode step of one layer (trigger, retrieve, store_cache, attention); one
        clustered launch on retrieval layers. q_all: [batch, Hq, d] (all heads)."""
        assert k_t.stride(0) == v_t.stride(0)
        self._chk(self._L.louiskv_decode_layer(self.h, layer, _ptr(q_all), q_all.stride(0), _ptr(k_t), _ptr(v_t),
                                               k_t.stride(0), _ptr(out), _ptr(out_f32), _ptr(flag_out),
                                               _ptr(r_out), _stream(stream)))

    # --- introspection ------------------------------------------------------
    def get_selection(self, layer, b, h):
        n = ctypes.c_int32()
        self._chk(self._L.louiskv_get_selection(self.h, layer, b, h, None, 0, ctypes.byref(n)))
        ids = np.zeros(max(n.value, 1), np.int32)
        self._chk(self._L.louiskv_get_selection(self.h, layer, b, h, ids.ctypes.data, ids.size, ctypes.byref(n)))
        return ids[:n.value].copy()

    def get_units(self, layer, b, h):
        n = ctypes.c_int32()
        self._chk(self._L.louiskv_get_units(self.h, layer, b, h, 0, None, None, None, ctypes.byref(n)))
        m = max(n.value, 1)
        cen = np.zeros((m, 128), np.float32)
        sizes = np.zeros(m, np.int32)
        first = np.zeros(m, np.int32)
        self._chk(self._L.louiskv_get_units(self.h, layer, b, h, m, cen.ctypes.data, sizes.ctypes.data,
                                            first.ctypes.data, ctypes.byref(n)))
        k = n.value
        return cen[:k].copy(), sizes[:k].copy(), first[:k].copy()

    def get_unit_positions(self, layer, b, h):
        n = ctypes.c_int64()
        self._chk(self._L.louiskv_get_unit_positions(self.h, layer, b, h, None, 0, ctypes.byref(n)))
        pos = np.zeros(max(n.value, 1), np.int32)
        self._chk(self._L.louiskv_get_unit_positions(self.h, layer, b, h, pos.ctypes.data, pos.size, ctypes.byref(n)))
        return pos[:n.value].copy()

    def get_working_set(self, layer, b, h):
        n = ctypes.c_int32()
        cap = max(self.cfg.budget_tokens, 1)
        K = np.zeros((cap, 128), np.uint16)
        V = np.zeros((cap, 128), np.uint16)
        self._chk(self._L.louiskv_get_working_set(self.h, layer, b, h, K.ctypes.data, V.ctypes.data, cap,
                                                  ctypes.byref(n)))
        return K[:n.value].copy(), V[:n.value].copy()

    def memory(self) -> dict:
        """Device bytes allocated by the context and pinned host-pool bytes (louiskv_get_memory)."""
        d, h = ctypes.c_uint64(), ctypes.c_uint64()
        self._chk(self._L.louiskv_get_memory(self.h, ctypes.byref(d), ctypes.byref(h)))
        return {"device_bytes": d.value, "host_pool_bytes": h.value}

    def set_prefill_timing(self, enable: bool = True):
        """Enable/disable (and reset) the cluster_prompt phase timer (louiskv_set_prefill_timing)."""
        self._chk(self._L.louiskv_set_prefill_timing(self.h, 1 if enable else 0))

    def prefill_times(self) -> dict:
        t = PrefillTimes()
        self._chk(self._L.louiskv_get_prefill_times(self.h, ctypes.byref(t)))
        return t.as_dict()

    def pool_numa_node(self) -> int:
        """NUMA node the pinned pool is bound to (-1: cudaHostAlloc, no binding)."""
        n = ctypes.c_int32()
        self._chk(self._L.louiskv_get_pool_numa_node(self.h, ctypes.byref(n)))
        return n.value

    def state_save(self, stream=None):
        """Checkpoint the decode state (device resident, stream ordered)."""
        self._chk(self._L.louiskv_state_save(self.h, _stream(stream)))

    def state_restore(self, stream=None):
        self._chk(self._L.louiskv_state_restore(self.h, _stream(stream)))

    def stats(self) -> dict:
        s = Stats()
        self._chk(self._L.louiskv_get_stats(self.h, ctypes.byref(s)))
        return s.as_dict()
