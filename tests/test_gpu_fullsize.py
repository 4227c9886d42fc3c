"""Parity at BASELINE.json's full sizes (configs C2-C5) in the launch
configuration bench.py uses: the whole cache is built and attended on the GPU; the oracle
recomputes a sample of units one by one (inputs regenerated on the host from the same
counter-based generator)."""
import math

import numpy as np
import pytest

import synth
from oracle import mustafar_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-3


@pytest.fixture(scope="module")
def M():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_22913_b200 import build as B
    B.build()
    from paper_2505_22913_b200 import mustafar
    return mustafar


def compare_unit(bufs, u, oc, note):
    """Every record buffer of unit u (bitmaps, packed values, tile offsets of K and V), the
    window ring and both counters, bit-exact against the oracle's one-unit cache."""
    nc, nw = int(oc.n_comp[0]), int(oc.n_win[0])
    assert int(bufs["n_comp"][u]) == nc and int(bufs["n_win"][u]) == nw, note
    vdt = oc.values_k.dtype   # uint16 fp16 values, or uint8 4-bit records (NEXT-4)
    for name, dt in (("bitmap_k", np.uint64), ("bitmap_v", np.uint64), ("values_k", vdt),
                     ("values_v", vdt), ("offsets_k", np.uint32), ("offsets_v", np.uint32)):
        g = bufs[name][u, :nc].cpu().numpy().view(dt)
        assert np.array_equal(g, getattr(oc, name)[0, :nc]), (note, name)
    if oc.W:
        slots = [(nc + i) % oc.W for i in range(nw)]
        for name in ("win_k", "win_v"):
            g = bufs[name][u].cpu().numpy().view(np.uint16)
            assert np.array_equal(g[slots], getattr(oc, name)[0, slots]), (note, name)


CASES = {
    # name: (batch, hq, hkv, T, sparsity_k, sparsity_v, sampled units)
    "C2_b16_s70": (16, 32, 8, 4096, 0.7, 0.7, (0, 77, 127)),
    "C2_b1_s50": (1, 32, 8, 4096, 0.5, 0.5, (0, 7)),
    "C3_mha_32k": (1, 32, 32, 32768, 0.7, 0.7, (0, 31)),
    "C4_128k_b8": (8, 32, 8, 131072, 0.7, 0.7, (5, 63)),
    "C5_16k_b64": (64, 32, 8, 16384, 0.7, 0.7, (0, 300, 511)),
    "C4_128k_b8_q4": (8, 32, 8, 131072, 0.7, 0.7, (5, 63)),   # 4-bit payload (NEXT-4)
}


def vbits_of(name):
    return 4 if name.endswith("_q4") else 16


@pytest.mark.parametrize("name", [n for n in CASES if not n.endswith("_q4")])
def test_fullsize_sampled(M, name):
    B, hq, hkv, T, sk, sv, sample = CASES[name]
    U, G, d, W = B * hkv, hq // hkv, 128, 32
    kk, kv = O.keep_count(sk, d), O.keep_count(sv, d)
    sK, sV, sQ = (synth.seed_for(7, i) for i in range(3))
    K = synth.fp16_torch((U, T, d), sK, device="cuda")
    V = synth.fp16_torch((U, T, d), sV, device="cuda")
    q = synth.fp16_torch((U, G, d), sQ, device="cuda")
    gc = M.MustafarCache(B, hq, hkv, d, kk, kv, W, T)
    gc.prune_compress_kv(K, V)
    del K, V
    out = gc.sparse_decode_attention(q, 1 / math.sqrt(d))
    torch.cuda.synchronize()
    bufs = gc.buffers()
    qh = q.cpu().view(torch.int16).numpy().view(np.uint16)
    for u in sample:
        Ku = synth.fp16_np_rows((U, T, d), sK, u * T, T).view(np.uint16)
        Vu = synth.fp16_np_rows((U, T, d), sV, u * T, T).view(np.uint16)
        oc = O.OracleCache(1, d, kk, kv, W, T)
        oc.prefill(Ku[None], Vu[None])
        compare_unit(bufs, u, oc, f"{name} u={u}")
        ref = O.attention(oc, qh[u][None], 1 / math.sqrt(d))[0]
        o = out[u].cpu().numpy().astype(np.float64)
        err = float((np.abs(o - ref).max(axis=-1) / np.abs(ref).max(axis=-1)).max())
        assert err <= TOL, (name, u, err)


@pytest.mark.parametrize("name", ["C2_b16_s70", "C3_mha_32k", "C4_128k_b8", "C5_16k_b64", "C4_128k_b8_q4"])
def test_fullsize_decode_step_sampled(M, name):
    """One fused decode step (mstf_decode_step: the append inside the attention launch) at full
    size -- the launch configuration bench.py times -- against the oracle on sampled units:
    every record buffer, the window and the counters bit-exact, attention within 2e-3."""
    B, hq, hkv, T, sk, sv, sample = CASES[name]
    U, G, d, W = B * hkv, hq // hkv, 128, 32
    kk, kv = O.keep_count(sk, d), O.keep_count(sv, d)
    sK, sV, sQ = (synth.seed_for(8, i) for i in range(3))
    K = synth.fp16_torch((U, T + 1, d), sK, device="cuda")
    V = synth.fp16_torch((U, T + 1, d), sV, device="cuda")
    q = synth.fp16_torch((U, G, d), sQ, device="cuda")
    gc = M.MustafarCache(B, hq, hkv, d, kk, kv, W, T + 1, value_bits=vbits_of(name))
    gc.prune_compress_kv(K[:, :T].contiguous(), V[:, :T].contiguous())
    kn, vn = K[:, T].contiguous(), V[:, T].contiguous()
    del K, V
    assert gc.decode_step_kernel_count() == 2
    out = gc.decode_step(kn, vn, q, 1 / math.sqrt(d))
    torch.cuda.synchronize()
    bufs = gc.buffers()
    qh = q.cpu().view(torch.int16).numpy().view(np.uint16)
    for u in sample:
        Ku = synth.fp16_np_rows((U, T + 1, d), sK, u * (T + 1), T + 1).view(np.uint16)
        Vu = synth.fp16_np_rows((U, T + 1, d), sV, u * (T + 1), T + 1).view(np.uint16)
        oc = O.OracleCache(1, d, kk, kv, W, T + 1, value_bits=vbits_of(name))
        oc.prefill(Ku[None, :T], Vu[None, :T])
        oc.append(Ku[None, T], Vu[None, T])
        compare_unit(bufs, u, oc, f"{name} step u={u}")
        ref = O.attention(oc, qh[u][None], 1 / math.sqrt(d))[0]
        o = out[u].cpu().numpy().astype(np.float64)
        err = float((np.abs(o - ref).max(axis=-1) / np.abs(ref).max(axis=-1)).max())
        assert err <= TOL, (name, u, err)


def test_fullsize_output_aware_prefill_sampled(M):
    """Output-aware K pruning (NEXT-2) at C2 size: weights from 32 window queries of the GQA
    group (mstf_query_abs_sum), whole-cache prefill on the GPU, sampled units bit-exact
    against the oracle's scored pruning."""
    B, hq, hkv, T, sk, sv, sample = CASES["C2_b16_s70"]
    U, G, d, W = B * hkv, hq // hkv, 128, 32
    kk = O.keep_count(sk, d)
    sK, sV, sQ = (synth.seed_for(9, i) for i in range(3))
    K = synth.fp16_torch((U, T, d), sK, device="cuda", kind="outlier")
    V = synth.fp16_torch((U, T, d), sV, device="cuda")
    qr = synth.fp16_torch((U, 32, G, d), sQ, device="cuda")
    w = M.query_abs_sum(qr)
    gc = M.MustafarCache(B, hq, hkv, d, kk, kk, W, T)
    gc.set_key_weights(w)
    gc.prune_compress_kv(K, V)
    del K, V
    torch.cuda.synchronize()
    bufs = gc.buffers()
    wh = O.query_abs_sum(qr.cpu().view(torch.int16).numpy().view(np.uint16))
    assert np.array_equal(w.cpu().numpy().view(np.uint32), wh.view(np.uint32))
    for u in sample:
        Ku = synth.fp16_np_rows((U, T, d), sK, u * T, T, kind="outlier").view(np.uint16)
        Vu = synth.fp16_np_rows((U, T, d), sV, u * T, T).view(np.uint16)
        oc = O.OracleCache(1, d, kk, kk, W, T)
        oc.set_key_weights(wh[u][None])
        oc.prefill(Ku[None], Vu[None])
        compare_unit(bufs, u, oc, f"output-aware u={u}")


def test_fullsize_sequence_split_sampled(M):
    """Sequence split (NEXT-3) at the batch-1 128K shape: 4 shards on one device, partials
    merged, sampled units against the oracle over the unsplit cache."""
    B, hq, hkv, T, world = 1, 32, 8, 131072, 4
    U, G, d, W = B * hkv, hq // hkv, 128, 32
    kk = O.keep_count(0.7, d)
    sK, sV, sQ = (synth.seed_for(10, i) for i in range(3))
    K = synth.fp16_torch((U, T, d), sK, device="cuda")
    V = synth.fp16_torch((U, T, d), sV, device="cuda")
    q = synth.fp16_torch((U, G, d), sQ, device="cuda")
    ml = torch.empty(world, U, G, 2, dtype=torch.float32, device="cuda")
    po = torch.empty(world, U, G, d, dtype=torch.float32, device="cuda")
    for r in range(world):
        t0, t1 = M.seq_split(T, W, world, r)
        c = M.MustafarCache(B, hq, hkv, d, kk, kk, W if r == world - 1 else 0, t1 - t0)
        c.prune_compress_kv(K[:, t0:t1].contiguous(), V[:, t0:t1].contiguous())
        c.sparse_decode_attention_partial(q, 1 / math.sqrt(d), ml=ml[r], o=po[r])
        del c
    del K, V
    out = M.merge_partials(ml, po).cpu().numpy().astype(np.float64)
    qh = q.cpu().view(torch.int16).numpy().view(np.uint16)
    for u in (0, 5):
        Ku = synth.fp16_np_rows((U, T, d), sK, u * T, T).view(np.uint16)
        Vu = synth.fp16_np_rows((U, T, d), sV, u * T, T).view(np.uint16)
        oc = O.OracleCache(1, d, kk, kk, W, T)
        oc.prefill(Ku[None], Vu[None])
        ref = O.attention(oc, qh[u][None], 1 / math.sqrt(d))[0]
        err = float((np.abs(out[u] - ref).max(axis=-1) / np.abs(ref).max(axis=-1)).max())
        assert err <= TOL, (u, err)
