"""C-ABI library: it loads without a GPU, exports every symbol include/mustafar.h declares,
and its host-side validation / sizing / mirror logic behaves (no kernel launches here)."""
import ctypes
import os
import re

import pytest

from paper_2505_22913_b200 import build as B
from paper_2505_22913_b200 import mustafar as M

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    B.build()
    return M.lib()


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "mustafar.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(mstf_[a-z_0-9]+)\s*\(", hdr)))


def test_exports_every_declared_symbol(L):
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(M.EXPORTS) == syms


def test_library_is_sm100a(L):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", M.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_keep_and_pad(L):
    assert L.mstf_keep_from_sparsity(0.7, 128) == 39
    assert L.mstf_keep_from_sparsity(0.5, 128) == 64
    assert L.mstf_keep_from_sparsity(0.0, 128) == 128
    assert L.mstf_keep_from_sparsity(1.0, 128) == -3
    assert [L.mstf_k_pad(k) for k in (1, 8, 9, 39, 64, 128)] == [8, 8, 16, 40, 64, 128]


def test_value_record_bytes(L):
    """R7 / R26: fp16 records are 2 * k_pad bytes; 4-bit records round_up(4 + ceil(k/2), 16)
    (the oracle's q4_record_bytes); any other width is rejected."""
    from oracle import mustafar_oracle as O
    for k in (1, 13, 39, 64, 127, 128):
        assert L.mstf_value_record_bytes(k, 16) == L.mstf_value_record_bytes(k, 0) == 2 * O.k_pad_of(k)
        assert L.mstf_value_record_bytes(k, 4) == O.q4_record_bytes(k)
    assert L.mstf_value_record_bytes(39, 8) == -1
    sizes = M.buffer_bytes(cfg(value_bits=4))
    assert sizes[M.BUFFERS.index("values_k")] == 4 * 100 * 32 + 16
    assert sizes[M.BUFFERS.index("values_v")] == 4 * 100 * 48 + 16
    assert L.mstf_cache_buffer_bytes(ctypes.byref(cfg(value_bits=5)), (ctypes.c_size_t * M.NUM_BUFFERS)()) == -1


def cfg(**kw):
    base = dict(batch=2, num_q_heads=8, num_kv_heads=2, head_dim=128, keep_k=39, keep_v=64, window=32,
                capacity=100, value_bits=16)
    base.update(kw)
    return M.Config(*[base[n] for n, _ in M.Config._fields_])


def test_buffer_bytes(L):
    sizes = M.buffer_bytes(cfg())
    U = 4
    guard = 16  # values buffers: tail guard for the attention kernels' per-token loads
    assert sizes == [U * 100 * 16, U * 100 * 16, U * 100 * 40 * 2 + guard, U * 100 * 64 * 2 + guard,
                     U * 100 * 8, U * 100 * 8, U * 32 * 128 * 2, U * 32 * 128 * 2, U * 4, U * 4]


@pytest.mark.parametrize("kw,code", [
    (dict(head_dim=100), -2), (dict(num_q_heads=7), -2), (dict(keep_k=0), -3), (dict(keep_v=129), -3),
    (dict(window=-1), -1), (dict(batch=0), -1)])
def test_config_validation(L, kw, code):
    sizes = (ctypes.c_size_t * M.NUM_BUFFERS)()
    assert L.mstf_cache_buffer_bytes(ctypes.byref(cfg(**kw)), sizes) == code


def _fake_cache(L, **kw):
    c = cfg(**kw)
    ptrs = (ctypes.c_void_p * M.NUM_BUFFERS)(*[0x10000 * (i + 1) for i in range(M.NUM_BUFFERS)])
    h = ctypes.c_void_p()
    st = L.mstf_cache_create(ctypes.byref(c), ptrs, ctypes.byref(h))
    return st, h


def test_create_rejects_unsupported_and_misaligned(L):
    assert _fake_cache(L, head_dim=256)[0] == -7
    assert _fake_cache(L, num_q_heads=32, num_kv_heads=2)[0] == -7   # G = 16 > 8
    c = cfg()
    ptrs = (ctypes.c_void_p * M.NUM_BUFFERS)(*[0x10008] * M.NUM_BUFFERS)
    assert L.mstf_cache_create(ctypes.byref(c), ptrs, ctypes.byref(ctypes.c_void_p())) == -1


def test_host_validation_before_launch(L):
    st, h = _fake_cache(L, capacity=10)
    assert st == 0
    try:
        # prefill longer than capacity + window -> ECAPACITY, no launch
        assert L.mstf_prune_compress_kv(h, ctypes.c_void_p(0x1000), ctypes.c_void_p(0x1000), 43, None, None) == -4
        # lengths out of range
        ln = (ctypes.c_int32 * 4)(1, 2, 3, 50)
        assert L.mstf_prune_compress_kv(h, ctypes.c_void_p(0x1000), ctypes.c_void_p(0x1000), 40, ln, None) == -1
        assert L.mstf_prune_compress_kv(h, ctypes.c_void_p(0x1000), ctypes.c_void_p(0x1000), -1, None, None) == -2
        # attention on an empty cache -> EEMPTY; too-small workspace -> EWORKSPACE
        ws = L.mstf_workspace_bytes(h)
        assert ws > 0
        q = ctypes.c_void_p(0x2000)
        assert L.mstf_sparse_decode_attention(h, q, 0.1, q, 0, ctypes.c_void_p(0x3000), ws - 1, None) == -8
        assert L.mstf_sparse_decode_attention(h, q, 0.1, q, 0, ctypes.c_void_p(0x3000), ws, None) == -5
        assert L.mstf_sparse_decode_attention(h, q, 0.1, q, 7, ctypes.c_void_p(0x3000), ws, None) == -1
        nc, nw = (ctypes.c_int32 * 4)(), (ctypes.c_int32 * 4)()
        assert L.mstf_cache_counts(h, nc, nw) == 0 and list(nc) == [0] * 4 and list(nw) == [0] * 4
        # output-aware key weights: 16-byte alignment, NULL resets; accumulator argument checks
        assert L.mstf_set_key_weights(h, ctypes.c_void_p(0x1004)) == -1
        assert L.mstf_set_key_weights(h, ctypes.c_void_p(0x1000)) == 0
        assert L.mstf_set_key_weights(h, None) == 0
        assert L.mstf_set_key_weights(None, None) == -1
        assert L.mstf_query_abs_sum(None, 4, 32, 4, 128, ctypes.c_void_p(0x1000), None) == -1
        assert L.mstf_query_abs_sum(ctypes.c_void_p(0x1000), 4, 32, 0, 128, ctypes.c_void_p(0x1000), None) == -1
        assert L.mstf_query_abs_sum(ctypes.c_void_p(0x1000), -1, 32, 4, 128, ctypes.c_void_p(0x1000), None) == -1
        # sequence split: partials need a 16-B aligned o and 8-B aligned ml; merge argument checks
        a = ctypes.c_void_p(0x4000)
        assert L.mstf_sparse_decode_attention_partial(h, q, 0.1, a, None, ctypes.c_void_p(0x3000), ws, None) == -1
        assert L.mstf_sparse_decode_attention_partial(h, q, 0.1, ctypes.c_void_p(0x4004), a,
                                                      ctypes.c_void_p(0x3000), ws, None) == -1
        assert L.mstf_merge_partials(0, 4, 4, 128, a, a, a, 0, None) == -1
        assert L.mstf_merge_partials(2, 4, 4, 128, a, a, a, 5, None) == -1
        assert L.mstf_merge_partials(2, 4, 4, 64, a, a, a, 0, None) == -7
        assert L.mstf_merge_partials(2, 4, 16, 128, a, a, a, 0, None) == -7
        t0, t1 = ctypes.c_int32(), ctypes.c_int32()
        assert L.mstf_seq_split(100, 32, 4, 4, ctypes.byref(t0), ctypes.byref(t1)) == -1
        assert L.mstf_seq_split(100, 32, 4, 3, ctypes.byref(t0), ctypes.byref(t1)) == 0 and t1.value == 100
    finally:
        L.mstf_cache_destroy(h)


@pytest.mark.parametrize("kk,kv,n", [(39, 39, 2), (32, 32, 2), (16, 16, 2), (64, 64, 2), (39, 64, 2), (128, 128, 2)])
def test_attention_kernel_count(L, kk, kv, n):
    """Every attention call is two launches: the attention kernel (register-staged stream-K or
    TMA-staged split grid, chosen by k_pad) and the split combine."""
    st, h = _fake_cache(L, keep_k=kk, keep_v=kv)
    assert st == 0
    try:
        assert L.mstf_attention_kernel_count(h) == n
    finally:
        L.mstf_cache_destroy(h)
    assert L.mstf_attention_kernel_count(None) == -1


def test_shard_units(L):
    got = [M.shard_units(512, 8, r) for r in range(8)]
    assert got == [(64 * r, 64 * (r + 1)) for r in range(8)]
    got = [M.shard_units(10, 4, r) for r in range(4)]
    assert got[0][0] == 0 and got[-1][1] == 10 and all(a[1] == b[0] for a, b in zip(got, got[1:]))
    with pytest.raises(M.MustafarError):
        M.shard_units(10, 0, 0)


def test_status_strings(L):
    for code in M.STATUS:
        assert L.mstf_status_string(code)
    assert b"sm_100a" in L.mstf_build_info()


def test_binding_refuses_cpu_tensors(L):
    import torch
    with pytest.raises(ValueError):
        M._dev_ptr(torch.zeros(4, dtype=torch.float16))
