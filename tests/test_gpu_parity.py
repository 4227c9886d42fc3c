"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs. Bit-exact for bitmaps / packed values / offsets / window / counters; attention
within ||o_gpu - o_ref||_inf / ||o_ref||_inf <= 2e-3 per (unit, head) (north star tolerance;
DESIGN.md R14)."""
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


def u16(t):
    return t.detach().cpu().view(torch.int16).numpy().view(np.uint16)


def compare_cache(gc, oc, note=""):
    b = gc.buffers()
    nc = b["n_comp"].cpu().numpy()
    nw = b["n_win"].cpu().numpy()
    assert nc.tolist() == oc.n_comp.tolist(), note
    assert nw.tolist() == oc.n_win.tolist(), note
    assert list(gc.counts()[0]) == oc.n_comp.tolist() and list(gc.counts()[1]) == oc.n_win.tolist()
    bmk = b["bitmap_k"].cpu().numpy().view(np.uint64)
    bmv = b["bitmap_v"].cpu().numpy().view(np.uint64)
    vk, vv = u16(b["values_k"]), u16(b["values_v"])
    ok_, ov_ = b["offsets_k"].cpu().numpy().view(np.uint32), b["offsets_v"].cpu().numpy().view(np.uint32)
    wk, wv = u16(b["win_k"]), u16(b["win_v"])
    for u in range(oc.U):
        n = int(nc[u])
        np.testing.assert_array_equal(bmk[u, :n], oc.bitmap_k[u, :n], err_msg=f"{note} bitmap_k u={u}")
        np.testing.assert_array_equal(bmv[u, :n], oc.bitmap_v[u, :n], err_msg=f"{note} bitmap_v u={u}")
        np.testing.assert_array_equal(vk[u, :n], oc.values_k[u, :n], err_msg=f"{note} values_k u={u}")
        np.testing.assert_array_equal(vv[u, :n], oc.values_v[u, :n], err_msg=f"{note} values_v u={u}")
        np.testing.assert_array_equal(ok_[u, :n], oc.offsets_k[u, :n], err_msg=f"{note} offsets_k u={u}")
        np.testing.assert_array_equal(ov_[u, :n], oc.offsets_v[u, :n], err_msg=f"{note} offsets_v u={u}")
        if oc.W:
            slots = [(n + i) % oc.W for i in range(int(nw[u]))]
            np.testing.assert_array_equal(wk[u, slots], oc.win_k[u, slots], err_msg=f"{note} win_k u={u}")
            np.testing.assert_array_equal(wv[u, slots], oc.win_v[u, slots], err_msg=f"{note} win_v u={u}")


def rel_err(o_gpu, o_ref):
    """max over (unit, head) of ||o_gpu - o_ref||_inf / ||o_ref||_inf."""
    d = np.abs(o_gpu.astype(np.float64) - o_ref).max(axis=-1)
    n = np.abs(o_ref).max(axis=-1)
    return float((d / n).max())


def make(M, U_b, hq, hkv, T, kk, kv, W, cap=None, kind="normal", seed=1, lengths=None):
    U = U_b * hkv
    K = synth.fp16_np((U, T, 128), synth.seed_for(seed, 0), kind)
    V = synth.fp16_np((U, T, 128), synth.seed_for(seed, 1), kind)
    cap = cap if cap is not None else max(T, 1)
    gc = M.MustafarCache(U_b, hq, hkv, 128, kk, kv, W, cap)
    oc = O.OracleCache(U, 128, kk, kv, W, cap)
    Kd = torch.from_numpy(K.view(np.int16)).cuda().view(torch.float16)
    Vd = torch.from_numpy(V.view(np.int16)).cuda().view(torch.float16)
    gc.prune_compress_kv(Kd, Vd, lengths=lengths)
    oc.prefill(K.view(np.uint16), V.view(np.uint16), lengths=lengths)
    torch.cuda.synchronize()
    return gc, oc


# --------------------------------------------------------------------------- K1 prefill / append
@pytest.mark.parametrize("kind", ["normal", "lattice", "zeros", "outlier"])
@pytest.mark.parametrize("kk,kv", [(39, 39), (64, 64), (13, 26), (128, 1), (1, 128)])
def test_prefill_bit_exact(M, kind, kk, kv):
    gc, oc = make(M, 2, 8, 2, 300, kk, kv, 32, kind=kind, seed=kk + 3 * kv)
    compare_cache(gc, oc, f"{kind} k={kk},{kv}")


@pytest.mark.parametrize("kk", [39, 64, 2])
def test_prefill_and_append_inf_nan_channels(M, kk):
    """Tokens with +-inf and NaN channels (R3: |x| is bits & 0x7FFF as an unsigned integer, so
    NaN patterns rank above inf, inf above every finite value). Records stay bit-exact with the
    oracle -- in particular exactly k channels kept per token, also when several NaNs sit in one
    token (the prefill's fp16-compare phase once undercounted them) or when k or more
    channels of a token are inf/NaN (the integer fallback)."""
    U_b, hkv, T = 1, 2, 80
    U = U_b * hkv
    K = synth.fp16_np((U, T + 4, 128), 4242)
    V = synth.fp16_np((U, T + 4, 128), 4243)
    rng = np.random.default_rng(kk)
    specials = np.array([0x7C00, 0xFC00, 0x7E00, 0xFE00, 0x7C01, 0x7FFF, 0x7D55], dtype=np.uint16)
    for arr in (K, V):
        a = arr.view(np.uint16)
        for u in range(U):
            for t in range(T + 4):
                n = [0, 1, 2, 3, 5, 40, 70][t % 7]   # 40 / 70 >= k for most k: integer fallback
                ch = rng.choice(128, size=n, replace=False)
                a[u, t, ch] = rng.choice(specials, size=n)
    gc = M.MustafarCache(U_b, 4, hkv, 128, kk, kk, 8, T + 4)
    oc = O.OracleCache(U, 128, kk, kk, 8, T + 4)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).cuda().view(torch.float16)
    gc.prune_compress_kv(dev(K[:, :T]), dev(V[:, :T]))
    oc.prefill(K[:, :T].view(np.uint16), V[:, :T].view(np.uint16))
    for i in range(4):
        gc.append_token(dev(K[:, T + i]), dev(V[:, T + i]))
        oc.append(K[:, T + i].view(np.uint16), V[:, T + i].view(np.uint16))
    torch.cuda.synchronize()
    compare_cache(gc, oc, f"inf/nan k={kk}")


@pytest.mark.parametrize("W", [0, 1, 5, 32, 64])
def test_prefill_windows_and_ragged(M, W):
    lengths = [0, 1, W, W + 1, 200, 137, 64, 3]
    gc, oc = make(M, 2, 8, 4, 200, 39, 64, W, lengths=lengths, seed=W)
    compare_cache(gc, oc, f"W={W}")


@pytest.mark.parametrize("W", [0, 1, 32])
def test_append_bit_exact_and_equals_long_prefill(M, W):
    U_b, hkv, T, n = 2, 2, 70, 45
    U = U_b * hkv
    K = synth.fp16_np((U, T + n, 128), 501 + W)
    V = synth.fp16_np((U, T + n, 128), 601 + W)
    gc = M.MustafarCache(U_b, 4, hkv, 128, 39, 39, W, T + n)
    oc = O.OracleCache(U, 128, 39, 39, W, T + n)
    Kd = torch.from_numpy(K.view(np.int16)).cuda().view(torch.float16)
    Vd = torch.from_numpy(V.view(np.int16)).cuda().view(torch.float16)
    gc.prune_compress_kv(Kd[:, :T].contiguous(), Vd[:, :T].contiguous())
    oc.prefill(K[:, :T].view(np.uint16), V[:, :T].view(np.uint16))
    for i in range(n):
        gc.append_token(Kd[:, T + i].contiguous(), Vd[:, T + i].contiguous())
        oc.append(K[:, T + i].view(np.uint16), V[:, T + i].view(np.uint16))
    torch.cuda.synchronize()
    compare_cache(gc, oc, f"append W={W}")
    # prefill(T) + n appends == prefill(T + n) on the GPU, byte for byte
    g2 = M.MustafarCache(U_b, 4, hkv, 128, 39, 39, W, T + n)
    g2.prune_compress_kv(Kd, Vd)
    torch.cuda.synchronize()
    b1, b2 = gc.buffers(), g2.buffers()
    nc = b1["n_comp"].cpu().numpy()
    for name in ("bitmap_k", "bitmap_v", "values_k", "values_v", "offsets_k", "offsets_v"):
        for u in range(U):
            assert torch.equal(b1[name][u, :nc[u]], b2[name][u, :nc[u]]), name
    assert torch.equal(b1["n_comp"], b2["n_comp"]) and torch.equal(b1["n_win"], b2["n_win"])


def test_append_capacity_error(M):
    gc = M.MustafarCache(1, 1, 1, 128, 39, 39, 0, 2)
    k = torch.zeros(1, 128, dtype=torch.float16, device="cuda")
    gc.append_token(k, k)
    gc.append_token(k, k)
    with pytest.raises(M.MustafarError):
        gc.append_token(k, k)


# --------------------------------------------------------------------------- K2/K3 attention
def check_attention(M, gc, oc, U_b, hq, hkv, seed, scale=None, qkind="normal", out_dtype=torch.float32):
    U, G = U_b * hkv, hq // hkv
    q = synth.fp16_np((U, G, 128), synth.seed_for(seed, 2), qkind)
    qd = torch.from_numpy(q.view(np.int16)).cuda().view(torch.float16)
    scale = 1 / math.sqrt(128) if scale is None else scale
    out = gc.sparse_decode_attention(qd, scale, out_dtype=out_dtype)
    torch.cuda.synchronize()
    ref = O.attention(oc, q.view(np.uint16), scale)
    err = rel_err(out.float().cpu().numpy(), ref)
    assert np.isfinite(out.float().cpu().numpy()).all()
    return err


@pytest.mark.parametrize("case", [
    # (batch, hq, hkv, T, keep_k, keep_v, W)
    (1, 1, 1, 64, 64, 64, 32),          # C1: 1 unit, 64 tokens, 50%
    (1, 1, 1, 64, 64, 64, 0),
    (2, 4, 4, 1000, 39, 39, 32),        # MHA, several chunks, ragged tail
    (2, 32, 8, 777, 39, 39, 32),        # GQA G=4
    (1, 8, 1, 3000, 64, 26, 32),        # G=8, K != V sparsity
    (1, 8, 1, 3000, 39, 39, 32),        # G=8, one unit: stream-K combine with 2 sub-warps per head
    (1, 1, 1, 3000, 39, 39, 32),        # G=1, one unit: combine with 4 sub-warps per head
    (3, 2, 1, 129, 128, 128, 32),       # sparsity 0 (dense through the sparse path)
    (1, 4, 2, 20, 39, 39, 32),          # window only (no compressed tokens)
    (2, 4, 2, 5000, 13, 13, 1),         # 90% sparsity, W = 1
])
def test_attention_matches_oracle(M, case):
    U_b, hq, hkv, T, kk, kv, W = case
    gc, oc = make(M, U_b, hq, hkv, T, kk, kv, W, seed=T + kk)
    err = check_attention(M, gc, oc, U_b, hq, hkv, seed=T)
    assert err <= TOL, err


def test_attention_ragged_units(M):
    lengths = [1, 31, 32, 33, 64, 65, 300, 1000]
    gc, oc = make(M, 2, 16, 4, 1000, 39, 39, 32, lengths=lengths, seed=77)
    assert check_attention(M, gc, oc, 2, 16, 4, seed=77) <= TOL


@pytest.mark.parametrize("case", [
    # (batch, hq, hkv, T, keep, W, lengths per unit or None)
    (16, 32, 8, 600, 39, 32, None),                                   # uniform: stream-K without prefix
    (3, 8, 2, 777, 39, 0, [777, 5, 300, 1, 64, 65]),                  # ragged, no window
    (64, 8, 2, 300, 39, 32, [(37 * i) % 300 + 1 for i in range(128)]),  # ragged, many units
    (2, 8, 2, 1000, 32, 32, [1000, 17, 16, 999]),                     # kpad 32 kernel
    (2, 8, 2, 1000, 16, 16, None),                                    # kpad 16 kernel
    (4, 16, 4, 700, 64, 64, [700, 5, 64, 333] * 4),                   # kpad 64 (50% sparsity)
])
def test_attention_schedules(M, case):
    """The stream-K schedule (units' blocks concatenated, worker ranges crossing unit
    boundaries; ragged caches through the device-side cost prefix) at several k_pad values,
    against the oracle."""
    U_b, hq, hkv, T, keep, W, lengths = case
    gc, oc = make(M, U_b, hq, hkv, T, keep, keep, W, lengths=lengths, seed=T + keep)
    assert check_attention(M, gc, oc, U_b, hq, hkv, seed=T) <= TOL


def test_attention_after_appends(M):
    U_b, hq, hkv, T, n = 1, 8, 2, 500, 40
    U = U_b * hkv
    K = synth.fp16_np((U, T + n, 128), 901)
    V = synth.fp16_np((U, T + n, 128), 902)
    gc = M.MustafarCache(U_b, hq, hkv, 128, 39, 39, 32, T + n)
    oc = O.OracleCache(U, 128, 39, 39, 32, T + n)
    Kd = torch.from_numpy(K.view(np.int16)).cuda().view(torch.float16)
    Vd = torch.from_numpy(V.view(np.int16)).cuda().view(torch.float16)
    gc.prune_compress_kv(Kd[:, :T].contiguous(), Vd[:, :T].contiguous())
    oc.prefill(K[:, :T].view(np.uint16), V[:, :T].view(np.uint16))
    for i in range(n):
        gc.append_token(Kd[:, T + i].contiguous(), Vd[:, T + i].contiguous())
        oc.append(K[:, T + i].view(np.uint16), V[:, T + i].view(np.uint16))
        if i % 13 == 0:
            assert check_attention(M, gc, oc, U_b, hq, hkv, seed=i) <= TOL


def test_attention_peaked_softmax_and_fp16_out(M):
    gc, oc = make(M, 1, 4, 1, 2000, 39, 39, 32, kind="outlier", seed=5)
    assert check_attention(M, gc, oc, 1, 4, 1, seed=5, scale=0.5) <= TOL
    assert check_attention(M, gc, oc, 1, 4, 1, seed=6, out_dtype=torch.float16) <= TOL


def test_attention_empty_unit_rejected(M):
    gc, _ = make(M, 1, 2, 2, 10, 39, 39, 32, lengths=[0, 10], seed=3)
    q = torch.zeros(2, 1, 128, dtype=torch.float16, device="cuda")
    with pytest.raises(M.MustafarError):
        gc.sparse_decode_attention(q)


# --------------------------------------------------------------------------- dense baseline
@pytest.mark.parametrize("U,G,T", [(1, 1, 64), (8, 4, 1000), (3, 8, 77)])
def test_dense_baseline_matches_oracle(M, U, G, T):
    K = synth.fp16_np((U, T, 128), 11)
    V = synth.fp16_np((U, T, 128), 12)
    q = synth.fp16_np((U, G, 128), 13)
    lengths = [T - (u % 3) for u in range(U)]
    dense = M.DenseAttention(U, G, 128, T)
    out = dense(torch.from_numpy(K.view(np.int16)).cuda().view(torch.float16),
                torch.from_numpy(V.view(np.int16)).cuda().view(torch.float16),
                torch.tensor(lengths, dtype=torch.int32, device="cuda"),
                torch.from_numpy(q.view(np.int16)).cuda().view(torch.float16), 1 / math.sqrt(128))
    torch.cuda.synchronize()
    ref = np.stack([O.attention_dense(q[u].view(np.uint16), K[u, :lengths[u]].view(np.uint16),
                                      V[u, :lengths[u]].view(np.uint16), 1 / math.sqrt(128)) for u in range(U)])
    assert rel_err(out.cpu().numpy(), ref) <= TOL


# --------------------------------------------------------------------------- fused decode step
def _twin_caches(M, U_b, hq, hkv, T, kk, kv, W, steps, lengths=None, seed=11):
    """Two GPU caches + one oracle cache with the same prefill, room for `steps` appends."""
    U = U_b * hkv
    K = synth.fp16_np((U, T + steps, 128), synth.seed_for(seed, 0))
    V = synth.fp16_np((U, T + steps, 128), synth.seed_for(seed, 1))
    cap = T + steps
    Kd = torch.from_numpy(K.view(np.int16)).cuda().view(torch.float16)
    Vd = torch.from_numpy(V.view(np.int16)).cuda().view(torch.float16)
    caches = []
    for _ in range(2):
        c = M.MustafarCache(U_b, hq, hkv, 128, kk, kv, W, cap)
        c.prune_compress_kv(Kd[:, :T].contiguous(), Vd[:, :T].contiguous(), lengths=lengths)
        caches.append(c)
    oc = O.OracleCache(U, 128, kk, kv, W, cap)
    oc.prefill(K[:, :T].view(np.uint16), V[:, :T].view(np.uint16), lengths=lengths)
    return caches, oc, K, V, Kd, Vd


@pytest.mark.parametrize("case", [
    # (batch, hq, hkv, T, keep_k, keep_v, W, steps, lengths)
    (16, 32, 8, 600, 39, 39, 32, 5, None),      # full window: every step evicts into a record
    (2, 8, 2, 10, 39, 39, 32, 30, None),        # window filling (no eviction), then evicting
    (2, 8, 2, 300, 39, 39, 0, 4, None),         # W = 0: the new token is compressed directly
    (1, 8, 1, 777, 32, 32, 32, 3, None),        # G = 8, k_pad 32
    (2, 8, 2, 400, 39, 39, 32, 3, [400, 37, 1, 64]),  # ragged: append + attention in sequence
    (1, 8, 2, 300, 64, 64, 32, 3, None),        # k_pad 64 (register kernel, vector loads): fused
    (1, 8, 2, 300, 26, 39, 32, 3, None),        # K != V sparsity (TMA kernel): unfused
    (200, 16, 8, 40, 39, 39, 32, 2, None),      # 1600 units > 1184 workers (appends loop)
    (2, 4, 4, 500, 39, 39, 32, 4, None),        # G = 1 (MHA, the C3 shape): fused
    (1, 1, 1, 3000, 39, 39, 32, 3, None),       # G = 1, one unit: fused, many workers per unit
    (3, 6, 3, 200, 39, 39, 32, 3, None),        # G = 2
])
def test_decode_step_equals_append_then_attention(M, case):
    U_b, hq, hkv, T, kk, kv, W, steps, lengths = case
    U, G = U_b * hkv, hq // hkv
    (cf, cs), oc, K, V, Kd, Vd = _twin_caches(M, U_b, hq, hkv, T, kk, kv, W, steps, lengths)
    scale = 1 / math.sqrt(128)
    for i in range(steps):
        q = synth.fp16_np((U, G, 128), synth.seed_for(500 + i, 2))
        qd = torch.from_numpy(q.view(np.int16)).cuda().view(torch.float16)
        kn, vn = Kd[:, T + i].contiguous(), Vd[:, T + i].contiguous()
        fused = lengths is None   # uniform cache: append inside the attention launch
        # fused: attention + combine; ragged: append + cost prefix + attention + combine
        assert cf.decode_step_kernel_count() == (2 if fused else 4)
        of = cf.decode_step(kn, vn, qd, scale)
        cs.append_token(kn, vn)
        os_ = cs.sparse_decode_attention(qd, scale)
        oc.append(K[:, T + i].view(np.uint16), V[:, T + i].view(np.uint16))
        torch.cuda.synchronize()
        # same plan, same arithmetic: the fused launch reproduces the two-call result exactly
        assert torch.equal(of, os_), (case, i, (of - os_).abs().max().item())
        assert rel_err(of.cpu().numpy(), O.attention(oc, q.view(np.uint16), scale)) <= TOL
    compare_cache(cf, oc, "fused")
    assert cf.counts() == cs.counts()


def test_decode_step_capacity_error(M):
    """A step that would compress past `capacity` is rejected before any launch, like append."""
    T, W = 40, 32
    K = torch.zeros(1, T, 128, dtype=torch.float16, device="cuda")
    c = M.MustafarCache(1, 4, 1, 128, 39, 39, W, T - W)  # compressed capacity exactly used by the prefill
    c.prune_compress_kv(K, K)
    q = torch.zeros(1, 4, 128, dtype=torch.float16, device="cuda")
    kn = torch.zeros(1, 128, dtype=torch.float16, device="cuda")
    with pytest.raises(M.MustafarError):
        c.decode_step(kn, kn, q)
    assert c.counts() == ([T - W], [W])
