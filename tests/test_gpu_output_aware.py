"""GPU parity of output-aware Key pruning (NEXT-2) through the C ABI against the
oracle: the float32 accumulator bit for bit, and prefill / append / fused decode-step records
bit for bit when the K channel weights are set (V stays magnitude pruned)."""
import math

import numpy as np
import pytest

import synth
from oracle import mustafar_oracle as O

from test_gpu_parity import M, compare_cache, rel_err, u16  # noqa: F401  (fixture + helpers)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.float16)


@pytest.mark.parametrize("U,R,G", [(1, 1, 1), (3, 32, 4), (8, 7, 1), (2, 32, 8), (4, 0, 2)])
def test_query_abs_sum_bit_exact(M, U, R, G):
    q = synth.fp16_np((U, R, G, 128), synth.seed_for(21, U * 100 + R), "normal", scale=3.0)
    w = M.query_abs_sum(dev(q))
    torch.cuda.synchronize()
    ref = O.query_abs_sum(q.view(np.uint16))
    assert np.array_equal(w.cpu().numpy().view(np.uint32), ref.view(np.uint32))


def weights(U, seed, kind="query"):
    if kind == "query":   # the paper's accumulator: 32 window queries x G = 4 heads
        q = synth.fp16_np((U, 32, 4, 128), seed)
        return O.query_abs_sum(q.view(np.uint16))
    if kind == "ties":    # few distinct weights -> many equal scores on lattice inputs
        rng = np.random.default_rng(seed)
        return rng.integers(0, 3, size=(U, 128)).astype(np.float32)
    if kind == "ones":
        return np.ones((U, 128), np.float32)
    raise ValueError(kind)


@pytest.mark.parametrize("kind,wkind", [("normal", "query"), ("outlier", "query"), ("lattice", "ties"),
                                        ("zeros", "ties"), ("normal", "ones")])
@pytest.mark.parametrize("kk", [39, 64, 13])
def test_prefill_output_aware_bit_exact(M, kind, wkind, kk):
    U_b, hkv, T, W = 2, 2, 300, 32
    U = U_b * hkv
    K = synth.fp16_np((U, T, 128), synth.seed_for(22, kk), kind)
    V = synth.fp16_np((U, T, 128), synth.seed_for(23, kk), kind)
    w = weights(U, synth.seed_for(24, kk), wkind)
    gc = M.MustafarCache(U_b, 8, hkv, 128, kk, 39, W, T)
    wd = torch.from_numpy(w).cuda()
    gc.set_key_weights(wd)
    gc.prune_compress_kv(dev(K), dev(V))
    oc = O.OracleCache(U, 128, kk, 39, W, T)
    oc.set_key_weights(w)
    oc.prefill(K.view(np.uint16), V.view(np.uint16))
    torch.cuda.synchronize()
    compare_cache(gc, oc, f"oa {kind}/{wkind} k={kk}")


@pytest.mark.parametrize("fused", [False, True])
def test_append_and_decode_step_output_aware(M, fused):
    """Weights change every step (the sliding window of the last 32 queries):
    evictions use the weights current at their step, on the GPU and in the oracle."""
    U_b, hq, hkv, T, n, W = 2, 8, 2, 64, 40, 32
    U, G = U_b * hkv, hq // hkv
    K = synth.fp16_np((U, T + n, 128), 31)
    V = synth.fp16_np((U, T + n, 128), 32)
    Q = synth.fp16_np((U, T + n, G, 128), 33)
    gc = M.MustafarCache(U_b, hq, hkv, 128, 39, 39, W, T + n)
    oc = O.OracleCache(U, 128, 39, 39, W, T + n)
    ring = np.zeros((U, 32, G, 128), np.float16)
    for i in range(32):                       # the prompt's last 32 queries
        ring[:, (T - 32 + i) % 32] = Q[:, T - 32 + i]
    wd = torch.empty(U, 128, dtype=torch.float32, device="cuda")
    gc.set_key_weights(wd)
    M.query_abs_sum(dev(ring), out=wd)
    oc.set_key_weights(O.query_abs_sum(ring.view(np.uint16)))
    gc.prune_compress_kv(dev(K[:, :T]), dev(V[:, :T]))
    oc.prefill(K[:, :T].view(np.uint16), V[:, :T].view(np.uint16))
    worst = 0.0
    for i in range(n):
        p = T + i
        ring[:, p % 32] = Q[:, p]            # the current query joins the window
        M.query_abs_sum(dev(ring), out=wd)
        oc.set_key_weights(O.query_abs_sum(ring.view(np.uint16)))
        q = dev(Q[:, p])
        if fused:
            out = gc.decode_step(dev(K[:, p]), dev(V[:, p]), q, 1 / math.sqrt(128))
        else:
            gc.append_token(dev(K[:, p]), dev(V[:, p]))
            out = gc.sparse_decode_attention(q, 1 / math.sqrt(128))
        oc.append(K[:, p].view(np.uint16), V[:, p].view(np.uint16))
        if i % 13 == 0 or i == n - 1:
            torch.cuda.synchronize()
            ref = O.attention(oc, Q[:, p].view(np.uint16), 1 / math.sqrt(128))
            worst = max(worst, rel_err(out.cpu().numpy(), ref))
    torch.cuda.synchronize()
    compare_cache(gc, oc, f"oa append fused={fused}")
    assert worst <= 2e-3, worst
