"""GPU parity of the sequence split through the C ABI: N shard caches on one
device (rank r ingests mstf_seq_split's token range; only the last shard keeps a window and
takes the decode appends), mstf_sparse_decode_attention_partial per shard, the shards' partials
stacked as an all-gather would, mstf_merge_partials -> O; compared with the oracle's attention
over the unsplit cache (<= 2e-3, R14), at several world sizes and after decode steps."""
import math

import numpy as np
import pytest

import synth
from oracle import mustafar_oracle as O

from test_gpu_parity import M, rel_err  # noqa: F401

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.float16)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("kk", [39, 64])
def test_seq_split_merge_matches_unsplit(M, world, kk):
    B_, hq, hkv, T, W, n = 1, 32, 8, 2000, 32, 20
    U, G = B_ * hkv, hq // hkv
    K = synth.fp16_np((U, T + n, 128), synth.seed_for(71, world), "outlier")
    V = synth.fp16_np((U, T + n, 128), synth.seed_for(72, world))
    Q = synth.fp16_np((n + 1, U, G, 128), synth.seed_for(73, world))
    shards = []
    for r in range(world):
        t0, t1 = M.seq_split(T, W, world, r)
        w = W if r == world - 1 else 0
        c = M.MustafarCache(B_, hq, hkv, 128, kk, kk, w, t1 - t0 + n + 1)
        c.prune_compress_kv(dev(K[:, t0:t1]), dev(V[:, t0:t1]))
        shards.append(c)
    oc = O.OracleCache(U, 128, kk, kk, W, T + n)
    oc.prefill(K[:, :T].view(np.uint16), V[:, :T].view(np.uint16))
    ml = torch.empty(world, U, G, 2, dtype=torch.float32, device="cuda")
    o = torch.empty(world, U, G, 128, dtype=torch.float32, device="cuda")
    worst = 0.0
    for i in range(n + 1):
        if i > 0:  # decode step: the new token goes to the last shard only
            p = T + i - 1
            shards[-1].append_token(dev(K[:, p]), dev(V[:, p]))
            oc.append(K[:, p].view(np.uint16), V[:, p].view(np.uint16))
        q = dev(Q[i])
        for r, c in enumerate(shards):
            c.sparse_decode_attention_partial(q, 1 / math.sqrt(128), ml=ml[r], o=o[r])
        out = M.merge_partials(ml, o)
        if i % 10 == 0:
            torch.cuda.synchronize()
            ref = O.attention(oc, Q[i].view(np.uint16), 1 / math.sqrt(128))
            worst = max(worst, rel_err(out.cpu().numpy(), ref))
    assert worst <= 2e-3, worst


def test_partial_matches_oracle_partial(M):
    """The partials themselves: m (log2 units) * ln 2 = the oracle's m, and o / l = the
    oracle's o / l (the shard's normalised attention)."""
    B_, hq, hkv, T, W = 2, 8, 2, 500, 32
    U, G = B_ * hkv, hq // hkv
    K = synth.fp16_np((U, T, 128), 81)
    V = synth.fp16_np((U, T, 128), 82)
    q = synth.fp16_np((U, G, 128), 83)
    c = M.MustafarCache(B_, hq, hkv, 128, 39, 39, W, T)
    c.prune_compress_kv(dev(K), dev(V))
    ml, o = c.sparse_decode_attention_partial(dev(q), 0.1)
    oc = O.OracleCache(U, 128, 39, 39, W, T)
    oc.prefill(K.view(np.uint16), V.view(np.uint16))
    m_ref, l_ref, o_ref = O.attention_partial(oc, q.view(np.uint16), 0.1)
    torch.cuda.synchronize()
    mlh, oh = ml.cpu().numpy().astype(np.float64), o.cpu().numpy().astype(np.float64)
    assert np.abs(mlh[..., 0] * math.log(2) - m_ref).max() <= 1e-4 * np.abs(m_ref).max()
    assert rel_err(oh / mlh[..., 1:2], o_ref / l_ref[..., None]) <= 2e-3


def test_merge_empty_and_f16(M):
    """m = -inf shards contribute nothing; an all-empty (unit, head) gives 0; fp16 output."""
    n, U, G = 3, 2, 4
    ml = torch.zeros(n, U, G, 2, device="cuda")
    o = torch.randn(n, U, G, 128, device="cuda")
    ml[..., 0] = -float("inf")
    ml[1, 0, :, 0] = 0.5
    ml[1, 0, :, 1] = 2.0
    out = M.merge_partials(ml, o, out_dtype=torch.float16)
    torch.cuda.synchronize()
    assert torch.allclose(out[0].float(), (o[1, 0] / 2.0), rtol=2e-3, atol=1e-3)
    assert torch.count_nonzero(out[1]) == 0


def test_seq_split_more_ranks_than_compressed_tokens(M):
    """T <= W: every compressed range is empty; those shards return the merge identity and
    the merge equals the unsplit attention (all tokens in the last shard's window)."""
    B_, hq, hkv, T, W, world = 1, 8, 2, 20, 32, 4
    U, G = B_ * hkv, hq // hkv
    K = synth.fp16_np((U, T, 128), 91)
    V = synth.fp16_np((U, T, 128), 92)
    q = synth.fp16_np((U, G, 128), 93)
    ml = torch.empty(world, U, G, 2, dtype=torch.float32, device="cuda")
    o = torch.empty(world, U, G, 128, dtype=torch.float32, device="cuda")
    for r in range(world):
        t0, t1 = M.seq_split(T, W, world, r)
        c = M.MustafarCache(B_, hq, hkv, 128, 39, 39, W if r == world - 1 else 0, max(t1 - t0, 1))
        if t1 > t0:
            c.prune_compress_kv(dev(K[:, t0:t1]), dev(V[:, t0:t1]))
        c.sparse_decode_attention_partial(dev(q), 0.1, ml=ml[r], o=o[r])
    out = M.merge_partials(ml, o).cpu().numpy()
    oc = O.OracleCache(U, 128, 39, 39, W, T)
    oc.prefill(K.view(np.uint16), V.view(np.uint16))
    assert rel_err(out, O.attention(oc, q.view(np.uint16), 0.1)) <= 2e-3
