"""CPU checks of the C ABI: the library loads, exports every symbol include/louiskv.h
declares, the ctypes structs match the C layout, and argument errors are synchronous."""
import ctypes
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "louiskv.h")


@pytest.fixture(scope="module")
def lkv():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2510_11292_b200 as m
    return m


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(louiskv_[a-z_]+)\s*\(", src)) - {"louiskv_status"})


def test_header_declares_binding_symbols(lkv):
    assert declared_functions() == sorted(lkv.SYMBOLS)


def test_library_exports_every_declared_symbol(lkv):
    out = subprocess.run(["nm", "-D", "--defined-only", lkv.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (louiskv_[a-z_]+)", out))
    missing = set(declared_functions()) - exported
    assert not missing, missing
    L = lkv.lib()
    for name in declared_functions():
        assert getattr(L, name) is not None
    assert "sm_100a" in lkv.version()


def test_ctypes_struct_layout_matches_c(lkv):
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "louiskv.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(louiskv_config), offsetof(louiskv_config, tau),
         offsetof(louiskv_config, full_cache_layers), offsetof(louiskv_config, device),
         sizeof(louiskv_stats), offsetof(louiskv_stats, segments_evicted), sizeof(louiskv_prefill_times),
         offsetof(louiskv_prefill_times, assign_flops), offsetof(louiskv_prefill_times, calls),
         offsetof(louiskv_config, fetch_mode), offsetof(louiskv_config, index_offload),
         offsetof(louiskv_config, pool_dtype), offsetof(louiskv_stats, dma_copies));
  return 0;
}
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        vals = list(map(int, subprocess.check_output([exe]).split()))
    C, S, T = lkv.Config, lkv.Stats, lkv.PrefillTimes
    assert vals == [ctypes.sizeof(C), C.tau.offset, C.full_cache_layers.offset, C.device.offset,
                    ctypes.sizeof(S), S.segments_evicted.offset, ctypes.sizeof(T), T.assign_flops.offset,
                    T.calls.offset, C.fetch_mode.offset, C.index_offload.offset, C.pool_dtype.offset,
                    S.dma_copies.offset]


def test_invalid_config_rejected_synchronously(lkv):
    L = lkv.lib()
    h = ctypes.c_void_p()
    bad = lkv.Config(num_layers=1, num_q_heads=1, num_kv_heads=1, head_dim=64, kv_head_count=1, max_batch=1,
                     max_prompt_len=16, max_output_len=4, window_tokens=4, avg_cluster_size=4)
    assert L.louiskv_create(ctypes.byref(bad), ctypes.byref(h)) == lkv.ERR_INVALID_ARG
    bad.head_dim = 128
    bad.num_q_heads = 3  # not a multiple of num_kv_heads... (3 % 1 == 0 but g=3 unsupported)
    assert L.louiskv_create(ctypes.byref(bad), ctypes.byref(h)) == lkv.ERR_INVALID_ARG
    assert L.louiskv_create(None, ctypes.byref(h)) == lkv.ERR_INVALID_ARG
    bad.num_q_heads = 128  # both trigger paths hold at most 64 query heads
    bad.num_kv_heads = 16
    assert L.louiskv_create(ctypes.byref(bad), ctypes.byref(h)) == lkv.ERR_INVALID_ARG
    bad.num_q_heads, bad.num_kv_heads = 4, 1
    bad.fetch_mode = 2  # only ZERO_COPY and BATCHED_DMA exist
    assert L.louiskv_create(ctypes.byref(bad), ctypes.byref(h)) == lkv.ERR_INVALID_ARG
    bad.fetch_mode = 0
    bad.index_offload = 2  # 0 (device index) or 1 (host index)
    assert L.louiskv_create(ctypes.byref(bad), ctypes.byref(h)) == lkv.ERR_INVALID_ARG
    bad.index_offload = 0
    bad.pool_dtype = 2  # BF16 or FP8_E4M3
    assert L.louiskv_create(ctypes.byref(bad), ctypes.byref(h)) == lkv.ERR_INVALID_ARG
    bad.pool_dtype, bad.fetch_mode = lkv.POOL_FP8_E4M3, lkv.FETCH_BATCHED_DMA  # copies cannot convert
    assert L.louiskv_create(ctypes.byref(bad), ctypes.byref(h)) == lkv.ERR_INVALID_ARG
    assert L.louiskv_state_restore(None, None) == lkv.ERR_INVALID_ARG
    assert L.louiskv_cluster_prompt(None, 0, None, None, 0, 0, 0, 1, 1, None) == lkv.ERR_INVALID_ARG


def test_no_cpu_fallback_without_gpu(lkv):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = lkv.lib()
    h = ctypes.c_void_p()
    ok = lkv.Config(num_layers=1, num_q_heads=1, num_kv_heads=1, head_dim=128, kv_head_count=1, max_batch=1,
                    max_prompt_len=16, max_output_len=4, window_tokens=4, avg_cluster_size=4)
    assert L.louiskv_create(ctypes.byref(ok), ctypes.byref(h)) == lkv.ERR_CUDA
