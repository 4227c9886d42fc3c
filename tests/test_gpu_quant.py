"""GPU parity of the prune-then-quantize payload: caches with
value_bits = 4 built by the CUDA kernels (bulk prefill, append, fused decode step) against the
oracle's records byte for byte, and decode attention over the quantized cache within 2e-3 of the
oracle's Algorithm 1 over the same reconstructed values."""
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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.float16)


def compare(gc, oc, note):
    b = gc.buffers()
    assert b["n_comp"].cpu().tolist() == oc.n_comp.tolist(), note
    assert b["n_win"].cpu().tolist() == oc.n_win.tolist(), note
    for u in range(oc.U):
        n = int(oc.n_comp[u])
        for name, dt in (("bitmap_k", np.uint64), ("bitmap_v", np.uint64), ("offsets_k", np.uint32),
                         ("offsets_v", np.uint32)):
            assert np.array_equal(b[name][u, :n].cpu().numpy().view(dt), getattr(oc, name)[u, :n]), (note, name, u)
        for name in ("values_k", "values_v"):
            g = b[name][u, :n].cpu().numpy()
            assert np.array_equal(g, getattr(oc, name)[u, :n]), (note, name, u)
        if oc.W:
            slots = [(n + i) % oc.W for i in range(int(oc.n_win[u]))]
            for name in ("win_k", "win_v"):
                g = b[name][u].cpu().numpy().view(np.uint16)
                assert np.array_equal(g[slots], getattr(oc, name)[u, slots]), (note, name, u)


def rel_err(o, ref):
    return float((np.abs(o.astype(np.float64) - ref).max(axis=-1) / np.abs(ref).max(axis=-1)).max())


@pytest.mark.parametrize("kind", ["normal", "lattice", "zeros", "outlier"])
@pytest.mark.parametrize("kk,kv", [(39, 39), (64, 64), (13, 26), (128, 1), (1, 128)])
def test_q4_prefill_and_appends_bit_exact(M, kind, kk, kv):
    U_b, hkv, T, n, W = 2, 2, 120, 40, 32
    U = U_b * hkv
    K = synth.fp16_np((U, T + n, 128), synth.seed_for(60 + kk, 0), kind)
    V = synth.fp16_np((U, T + n, 128), synth.seed_for(60 + kv, 1), kind)
    gc = M.MustafarCache(U_b, 8, hkv, 128, kk, kv, W, T + n, value_bits=4)
    oc = O.OracleCache(U, 128, kk, kv, W, T + n, value_bits=4)
    gc.prune_compress_kv(dev(K[:, :T]), dev(V[:, :T]))
    oc.prefill(K[:, :T].view(np.uint16), V[:, :T].view(np.uint16))
    torch.cuda.synchronize()
    compare(gc, oc, f"prefill {kind} {kk},{kv}")
    for i in range(n):
        gc.append_token(dev(K[:, T + i]), dev(V[:, T + i]))
        oc.append(K[:, T + i].view(np.uint16), V[:, T + i].view(np.uint16))
    torch.cuda.synchronize()
    compare(gc, oc, f"append {kind} {kk},{kv}")


@pytest.mark.parametrize("W", [0, 5, 32])
@pytest.mark.parametrize("kk,kv", [(39, 39), (64, 8)])
def test_q4_bulk_prefill_ragged(M, W, kk, kv):
    """The 4-bit payload through the bulk prefill kernel (k <= 64: one code word per lane of the
    token's eight) on ragged units: lengths 0, 1, W, W + 1 and long ones across the kernel's
    4-token groups and 32-token warp spans; every record buffer bit-exact (R25-R26)."""
    U_b, hkv, T = 2, 4, 300
    U = U_b * hkv
    lengths = [0, 1, W, W + 1, 300, 137, 64, 33]
    K = synth.fp16_np((U, T, 128), synth.seed_for(90 + W, kk), "normal")
    V = synth.fp16_np((U, T, 128), synth.seed_for(91 + W, kv), "lattice")
    gc = M.MustafarCache(U_b, 8, hkv, 128, kk, kv, W, T, value_bits=4)
    oc = O.OracleCache(U, 128, kk, kv, W, T, value_bits=4)
    gc.prune_compress_kv(dev(K), dev(V), lengths=lengths)
    oc.prefill(K.view(np.uint16), V.view(np.uint16), lengths=lengths)
    torch.cuda.synchronize()
    compare(gc, oc, f"ragged W={W} {kk},{kv}")


@pytest.mark.parametrize("case", [
    # (batch, hq, hkv, T, keep_k, keep_v, W, lengths)
    (1, 1, 1, 64, 64, 64, 32, None),
    (2, 32, 8, 777, 39, 39, 32, None),       # G = 4
    (2, 4, 4, 1000, 39, 39, 32, None),       # G = 1
    (1, 8, 1, 3000, 64, 26, 32, None),       # G = 8, K != V sparsity
    (2, 8, 2, 600, 39, 39, 0, [600, 5, 300, 1]),   # ragged, no window
    (1, 4, 2, 20, 39, 39, 32, None),         # window only
])
def test_q4_attention_matches_oracle(M, case):
    U_b, hq, hkv, T, kk, kv, W, lengths = case
    U, G = U_b * hkv, hq // hkv
    K = synth.fp16_np((U, T, 128), synth.seed_for(T, 0))
    V = synth.fp16_np((U, T, 128), synth.seed_for(T, 1))
    q = synth.fp16_np((U, G, 128), synth.seed_for(T, 2))
    gc = M.MustafarCache(U_b, hq, hkv, 128, kk, kv, W, max(T, 1), value_bits=4)
    oc = O.OracleCache(U, 128, kk, kv, W, max(T, 1), value_bits=4)
    gc.prune_compress_kv(dev(K), dev(V), lengths=lengths)
    oc.prefill(K.view(np.uint16), V.view(np.uint16), lengths=lengths)
    out = gc.sparse_decode_attention(dev(q), 1 / math.sqrt(128))
    torch.cuda.synchronize()
    compare(gc, oc, f"attn {case}")
    ref = O.attention(oc, q.view(np.uint16), 1 / math.sqrt(128))
    assert rel_err(out.cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("case", [(16, 32, 8, 600, 39, 32, 4), (2, 8, 2, 10, 39, 32, 30), (2, 4, 4, 300, 64, 0, 3)])
def test_q4_decode_step_matches_oracle(M, case):
    """The fused decode step on a quantized cache: append (evicting into a 4-bit record) inside the
    attention launch, step after step, against the oracle."""
    U_b, hq, hkv, T, keep, W, steps = case
    U, G = U_b * hkv, hq // hkv
    K = synth.fp16_np((U, T + steps, 128), synth.seed_for(90, 0))
    V = synth.fp16_np((U, T + steps, 128), synth.seed_for(90, 1))
    gc = M.MustafarCache(U_b, hq, hkv, 128, keep, keep, W, T + steps, value_bits=4)
    oc = O.OracleCache(U, 128, keep, keep, W, T + steps, value_bits=4)
    gc.prune_compress_kv(dev(K[:, :T]), dev(V[:, :T]))
    oc.prefill(K[:, :T].view(np.uint16), V[:, :T].view(np.uint16))
    for i in range(steps):
        q = synth.fp16_np((U, G, 128), synth.seed_for(700 + i, 2))
        assert gc.decode_step_kernel_count() == 2
        out = gc.decode_step(dev(K[:, T + i]), dev(V[:, T + i]), dev(q), 1 / math.sqrt(128))
        oc.append(K[:, T + i].view(np.uint16), V[:, T + i].view(np.uint16))
        torch.cuda.synchronize()
        assert rel_err(out.cpu().numpy(), O.attention(oc, q.view(np.uint16), 1 / math.sqrt(128))) <= TOL
    compare(gc, oc, f"step {case}")
