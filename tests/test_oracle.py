"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: values the paper or
SPEC print (tests/golden/spec_examples.json), closed forms, brute force on tiny inputs,
invariants, and reductions to library routines (torch SDPA in float64)."""
import itertools
import json
import math
import os

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import synth
from oracle import mustafar_oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def bits_of(vals):
    return np.asarray(vals, dtype=np.float16).view(np.uint16)


# ----------------------------------------------------------------------------- pruning
def test_keep_counts_closed_form():
    for d, s, k in GOLD["keep_counts"]["cases"]:
        assert O.keep_count(s, d) == k


def test_keep_count_rejects_bad_sparsity():
    with pytest.raises(ValueError):
        O.keep_count(1.0, 128)
    with pytest.raises(ValueError):
        O.keep_count(-0.1, 128)


def test_spec_prune_example():
    g = GOLD["prune_row"]
    assert O.prune_tokens(bits_of(g["row"]), g["k"]).tolist() == g["keep"]


def test_spec_prune_ties_and_signed_zero():
    g = GOLD["prune_ties"]
    assert O.prune_tokens(bits_of(g["row"]), g["k"]).tolist() == g["keep"]


def _brute_keep(row_bits, k):
    """O(d^2) rank count: keep c iff fewer than k channels beat it under (mag, index)."""
    mag = [int(b) & 0x7FFF for b in row_bits]
    d = len(mag)
    return [sum(1 for c2 in range(d) if (mag[c2], c2) > (mag[c], c)) < k for c in range(d)]


@pytest.mark.parametrize("kind", ["normal", "lattice", "zeros"])
@pytest.mark.parametrize("k", [1, 13, 39, 64, 127, 128])
def test_prune_matches_bruteforce_rank(kind, k):
    X = synth.fp16_np((24, 128), synth.seed_for(9, k), kind).view(np.uint16)
    keep = O.prune_tokens(X, k)
    assert (keep.sum(axis=1) == k).all()
    for t in range(X.shape[0]):
        assert keep[t].tolist() == _brute_keep(X[t], k)


def test_prune_exhaustive_subsets_d8():
    """The kept set maximises sum|x| over all k-subsets; among maximisers it is the one
    the tie rule selects (every kept channel beats every pruned one under (mag, index))."""
    rng = np.random.default_rng(0)
    for trial in range(300):
        row = rng.integers(-3, 4, size=8).astype(np.float16) * np.float16(0.5)
        b = row.view(np.uint16)
        mag = (b & 0x7FFF).astype(np.int64)
        k = int(rng.integers(1, 9))
        keep = O.prune_tokens(b, k)
        best = max(sum(mag[list(s)]) for s in itertools.combinations(range(8), k))
        assert mag[keep].sum() == best
        kept = np.flatnonzero(keep)
        pruned = np.flatnonzero(~keep)
        for c in kept:
            for c2 in pruned:
                assert (mag[c], c) > (mag[c2], c2)


@settings(max_examples=60, deadline=None)
@given(st.lists(st.integers(0, 0xFFFF).filter(lambda v: (v & 0x7C00) != 0x7C00), min_size=64, max_size=64),
       st.integers(1, 64))
def test_prune_property_d64(words, k):
    b = np.array(words, dtype=np.uint16)
    assert O.prune_tokens(b, k).tolist() == _brute_keep(b, k)


def test_sparsity_zero_keeps_all():
    X = synth.fp16_np((5, 128), 3).view(np.uint16)
    assert O.prune_tokens(X, O.keep_count(0.0, 128)).all()


# ----------------------------------------------------------------------------- format
def test_compress_two_ends_golden():
    g = GOLD["compress_two_ends"]
    row = np.zeros(g["d"], np.float16)
    for c, v in g["nonzero"].items():
        row[int(c)] = v
    b = row.view(np.uint16)[None]
    keep = O.prune_tokens(b, g["k"])
    bm, vals, offs = O.compress_tokens(b, keep, g["k"])
    assert [f"{int(x):016x}" for x in bm[0]] == g["bitmap_hex"]
    assert vals[0].view(np.float16).astype(float).tolist() == g["values"]
    assert offs[0].tolist() == g["offsets"]


@pytest.mark.parametrize("d", [64, 128, 256])
@pytest.mark.parametrize("s", [0.0, 0.3, 0.5, 0.7, 0.9])
@pytest.mark.parametrize("kind", ["normal", "zeros", "lattice"])
def test_round_trip_lossless(d, s, kind):
    """decompress(compress(x)) == pruned x bit-exactly."""
    k = O.keep_count(s, d)
    X = synth.fp16_np((40, d), 77, kind).view(np.uint16)
    keep = O.prune_tokens(X, k)
    bm, vals, offs = O.compress_tokens(X, keep, k, first_record=5)
    assert (np.array([bin(int(w)).count("1") for w in bm.reshape(-1)]).reshape(bm.shape).sum(1) == k).all()
    assert (vals[:, k:] == 0).all()
    back = O.decompress_tokens(bm, vals, offs, k, d, first_record=5)
    assert np.array_equal(back, O.apply_keep(X, keep))


def test_offsets_are_prefix_counts():
    X = synth.fp16_np((7, 128), 5).view(np.uint16)
    k = 39
    keep = O.prune_tokens(X, k)
    bm, vals, offs = O.compress_tokens(X, keep, k, first_record=3)
    for t in range(7):
        n0 = int(keep[t, :64].sum())
        assert offs[t].tolist() == [(3 + t) * 40, (3 + t) * 40 + n0]
        assert vals[t, :k].tolist() == X[t][keep[t]].tolist()
        for j in range(2):
            word = int(bm[t, j])
            assert [(word >> i) & 1 for i in range(64)] == keep[t, 64 * j: 64 * j + 64].astype(int).tolist()


def test_decompress_detects_corruption():
    X = synth.fp16_np((4, 128), 6).view(np.uint16)
    keep = O.prune_tokens(X, 39)
    bm, vals, offs = O.compress_tokens(X, keep, 39)
    bad = bm.copy()
    bad[1, 0] ^= np.uint64(1 << 5)
    with pytest.raises(O.FormatError):
        O.decompress_tokens(bad, vals, offs, 39, 128)
    badv = vals.copy()
    badv[2, 39] = 1
    with pytest.raises(O.FormatError):
        O.decompress_tokens(bm, badv, offs, 39, 128)
    bado = offs.copy()
    bado[0, 1] += 1
    with pytest.raises(O.FormatError):
        O.decompress_tokens(bm, vals, bado, 39, 128)


def test_tile_byte_model_golden():
    for nnz, nbytes in GOLD["tile_bytes"]["cases"]:
        assert int(O._pad8(nnz)) * 2 + 8 + 4 == nbytes


def test_compression_ratio_matches_paper():
    """P:441 compression ratios, reproduced by the paper-orientation byte model on
    synthetic normal KV (T = 2048 + 256 tokens, W = 32)."""
    g = GOLD["compression_ratio"]
    T, d = 2304, 128
    K = synth.fp16_np((T, d), 1).view(np.uint16)
    V = synth.fp16_np((T, d), 2).view(np.uint16)
    for sk, sv, want in g["cases"]:
        kk = O.prune_tokens(K, O.keep_count(sk, d)) if sk is not None else None
        kv = O.prune_tokens(V, O.keep_count(sv, d)) if sv is not None else None
        c, dn = O.size_model_paper(kk, kv)
        assert abs(c / dn - want) <= g["tolerance"], (sk, sv, c / dn, want)


def test_build_layout_bytes():
    # 70%: record = 16 B bitmap + 80 B values (+ 8 B offsets) vs 256 B dense per token
    c, dn = O.size_model_build(1032, 128, 39, 39, W=32, with_offsets=False)
    assert c == 2 * (1000 * 96 + 32 * 256) and dn == 2 * 1032 * 256


# ----------------------------------------------------------------------------- cache
def test_prefill_counts_golden():
    g = GOLD["prefill_counts"]
    for T, nc, nw in g["cases"]:
        c = O.OracleCache(1, 128, 64, 64, g["window"], capacity=max(T, 1))
        X = synth.fp16_np((1, T, 128), T).view(np.uint16)
        c.prefill(X, X)
        assert (c.n_comp[0], c.n_win[0]) == (nc, nw)


@pytest.mark.parametrize("W", [0, 1, 32])
def test_prefill_plus_appends_equals_longer_prefill(W):
    U, T, n, d = 3, 50, 40, 128
    K = synth.fp16_np((U, T + n, d), 11).view(np.uint16)
    V = synth.fp16_np((U, T + n, d), 12).view(np.uint16)
    a = O.OracleCache(U, d, 39, 64, W, capacity=T + n)
    a.prefill(K[:, :T], V[:, :T])
    for i in range(n):
        a.append(K[:, T + i], V[:, T + i])
    b = O.OracleCache(U, d, 39, 64, W, capacity=T + n)
    b.prefill(K, V)
    for name in ("bitmap_k", "bitmap_v", "values_k", "values_v", "offsets_k", "offsets_v",
                 "win_k", "win_v", "n_comp", "n_win"):
        assert np.array_equal(getattr(a, name), getattr(b, name)), name


def test_window_tokens_bit_identical():
    """the most recent W tokens are bit-identical to their originals."""
    U, T, d, W = 2, 90, 128, 32
    K = synth.fp16_np((U, T, d), 21).view(np.uint16)
    c = O.OracleCache(U, d, 39, 39, W, capacity=T)
    c.prefill(K, K)
    for u in range(U):
        kc, vc, kl, vl = c.tokens(u)
        assert np.array_equal(kl, K[u, T - W:])
        assert np.array_equal(kc, O.apply_keep(K[u, :T - W], O.prune_tokens(K[u, :T - W], 39)))


def test_ragged_lengths():
    U, T, d = 4, 70, 128
    K = synth.fp16_np((U, T, d), 31).view(np.uint16)
    c = O.OracleCache(U, d, 64, 64, 32, capacity=T)
    c.prefill(K, K, lengths=[0, 1, 33, 70])
    assert c.n_comp.tolist() == [0, 0, 1, 38] and c.n_win.tolist() == [0, 1, 32, 32]


def test_capacity_overflow():
    c = O.OracleCache(1, 128, 64, 64, 0, capacity=2)
    X = synth.fp16_np((1, 3, 128), 1).view(np.uint16)
    with pytest.raises(OverflowError):
        c.prefill(X, X)


# ----------------------------------------------------------------------------- attention
def _sdpa64(q, K, V, scale):
    import torch
    qt = torch.from_numpy(O.fp16_to_f64(q))[None, :, None, :]          # [1, G, 1, d]
    kt = torch.from_numpy(O.fp16_to_f64(K))[None, None].expand(1, q.shape[0], -1, -1)
    vt = torch.from_numpy(O.fp16_to_f64(V))[None, None].expand(1, q.shape[0], -1, -1)
    o = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, scale=scale)
    return o[0, :, 0, :].numpy()


def test_sparsity_zero_equals_sdpa_float64():
    """S:440 / S:428: with nothing pruned, Alg. 1 is textbook attention (library SDPA)."""
    U, T, d, G = 2, 77, 128, 4
    K = synth.fp16_np((U, T, d), 41).view(np.uint16)
    V = synth.fp16_np((U, T, d), 42).view(np.uint16)
    q = synth.fp16_np((U, G, d), 43).view(np.uint16)
    c = O.OracleCache(U, d, 128, 128, 32, capacity=T)
    c.prefill(K, V)
    out = O.attention(c, q, 1 / math.sqrt(d))
    for u in range(U):
        np.testing.assert_allclose(out[u], _sdpa64(q[u], K[u], V[u], 1 / math.sqrt(d)), rtol=1e-12, atol=1e-14)


def test_pruned_attention_equals_sdpa_on_zero_filled():
    """Central equivalence: compressed Alg. 1 == dense attention over the zero-filled
    pruned K/V (window rows unpruned)."""
    U, T, d, G, W = 2, 120, 128, 2, 32
    K = synth.fp16_np((U, T, d), 51).view(np.uint16)
    V = synth.fp16_np((U, T, d), 52).view(np.uint16)
    q = synth.fp16_np((U, G, d), 53).view(np.uint16)
    c = O.OracleCache(U, d, 39, 64, W, capacity=T)
    c.prefill(K, V)
    out = O.attention(c, q, 0.1)
    for u in range(U):
        Kp = K[u].copy(); Vp = V[u].copy()
        Kp[:T - W] = O.apply_keep(K[u, :T - W], O.prune_tokens(K[u, :T - W], 39))
        Vp[:T - W] = O.apply_keep(V[u, :T - W], O.prune_tokens(V[u, :T - W], 64))
        np.testing.assert_allclose(out[u], _sdpa64(q[u], Kp, Vp, 0.1), rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("n,G", [(1, 1), (64, 4), (333, 8)])
def test_attention_dense_equals_sdpa_float64(n, G):
    """attention_dense (the checker of the dense-KV baseline kernel) is textbook attention:
    pinned to torch SDPA in float64 (a library routine), including n = 1 (-> v0)."""
    d = 128
    K = synth.fp16_np((n, d), 71 + n).view(np.uint16)
    V = synth.fp16_np((n, d), 72 + n).view(np.uint16)
    q = synth.fp16_np((G, d), 73 + n).view(np.uint16)
    for scale in (1 / math.sqrt(d), 0.7):
        np.testing.assert_allclose(O.attention_dense(q, K, V, scale), _sdpa64(q, K, V, scale),
                                   rtol=1e-12, atol=1e-14)
    if n == 1:
        assert np.array_equal(O.attention_dense(q, K, V, 0.1), np.broadcast_to(O.fp16_to_f64(V[0]), (G, d)))


@pytest.mark.parametrize("W", [0, 5, 400])
def test_attention_dense_equals_cache_attention_unpruned(W):
    """With keep = d nothing is pruned, so Alg. 1 over the compressed cache (any window,
    including W >= T: all tokens dense) equals attention_dense over the raw K/V."""
    U, T, d, G = 2, 130, 128, 4
    K = synth.fp16_np((U, T, d), 81).view(np.uint16)
    V = synth.fp16_np((U, T, d), 82).view(np.uint16)
    q = synth.fp16_np((U, G, d), 83).view(np.uint16)
    c = O.OracleCache(U, d, d, d, W, capacity=T)
    c.prefill(K, V)
    out = O.attention(c, q, 1 / math.sqrt(d))
    for u in range(U):
        np.testing.assert_allclose(out[u], O.attention_dense(q[u], K[u], V[u], 1 / math.sqrt(d)),
                                   rtol=1e-12, atol=1e-14)


def test_attention_dense_shift_and_permutation():
    """Invariants of softmax(scale q K^T) V that a transposed operand or a normalisation over
    the wrong axis would break: scale 0 gives the mean of V for every head, and permuting the
    tokens (K and V rows together) leaves the output unchanged."""
    n, d, G = 50, 128, 2
    K = synth.fp16_np((n, d), 91).view(np.uint16)
    V = synth.fp16_np((n, d), 92).view(np.uint16)
    q = synth.fp16_np((G, d), 93).view(np.uint16)
    np.testing.assert_allclose(O.attention_dense(q, K, V, 0.0),
                               np.broadcast_to(O.fp16_to_f64(V).mean(axis=0), (G, d)), rtol=1e-13, atol=1e-15)
    perm = np.random.default_rng(3).permutation(n)
    np.testing.assert_allclose(O.attention_dense(q, K[perm], V[perm], 0.3), O.attention_dense(q, K, V, 0.3),
                               rtol=1e-12, atol=1e-14)


def test_spmv_score_golden():
    g = GOLD["spmv_score"]
    row = np.zeros(g["d"], np.float16)
    for c, v in g["token"].items():
        row[int(c)] = v
    b = row.view(np.uint16)[None]
    keep = O.prune_tokens(b, g["k"])
    bm, vals, offs = O.compress_tokens(b, keep, g["k"])
    kc = O.decompress_tokens(bm, vals, offs, g["k"], g["d"])
    q = np.ones(g["d"], np.float16).view(np.uint16)
    assert float(O.fp16_to_f64(kc[0]) @ O.fp16_to_f64(q)) == g["score"]


def test_weighted_values_golden():
    g = GOLD["weighted_values"]
    q = np.zeros((1, 2), np.float16).view(np.uint16)
    K = np.ones((2, 2), np.float16).view(np.uint16)
    V = np.array([g["v0"], g["v1"]], np.float16).view(np.uint16)
    out = O.attention_regions(q, np.zeros((0, 2), np.uint16), np.zeros((0, 2), np.uint16), K, V, 1.0)
    assert out[0].tolist() == g["out"]


def test_single_token_returns_v0():
    d = 128
    K = synth.fp16_np((1, 1, d), 61).view(np.uint16)
    V = synth.fp16_np((1, 1, d), 62).view(np.uint16)
    q = synth.fp16_np((1, 4, d), 63).view(np.uint16)
    for W in (0, 32):
        c = O.OracleCache(1, d, 39, 39, W, capacity=1)
        c.prefill(K, V)
        out = O.attention(c, q, 0.088)
        vhat = O.fp16_to_f64(c.tokens(0)[1] if W == 0 else V[0])[0]
        for g in range(4):
            assert np.array_equal(out[0, g], vhat)


def test_zero_query_gives_mean_of_values():
    U, T, d, W = 1, 64, 128, 32
    K = synth.fp16_np((U, T, d), 71).view(np.uint16)
    V = synth.fp16_np((U, T, d), 72).view(np.uint16)
    c = O.OracleCache(U, d, 39, 39, W, capacity=T)
    c.prefill(K, V)
    out = O.attention(c, np.zeros((1, 1, d), np.uint16), 0.088)
    kc, vc, kl, vl = c.tokens(0)
    mean = np.concatenate([O.fp16_to_f64(vc), O.fp16_to_f64(vl)]).mean(axis=0)
    np.testing.assert_allclose(out[0, 0], mean, rtol=1e-13, atol=1e-15)


def test_permutation_invariance_and_gqa_identical_queries():
    d = 128
    KC = synth.fp16_np((50, d), 81).view(np.uint16)
    VC = synth.fp16_np((50, d), 82).view(np.uint16)
    q1 = synth.fp16_np((1, d), 83).view(np.uint16)
    q = np.repeat(q1, 4, axis=0)
    e = np.zeros((0, d), np.uint16)
    a = O.attention_regions(q, KC, VC, e, e, 0.09)
    perm = np.random.default_rng(1).permutation(50)
    b = O.attention_regions(q, KC[perm[:30]], VC[perm[:30]], KC[perm[30:]], VC[perm[30:]], 0.09)
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-15)
    for g in range(1, 4):
        assert np.array_equal(a[0], a[g])


def test_needle_dominates():
    """A key aligned with q and a large scale puts ~all weight on that token."""
    d = 128
    K = synth.fp16_np((40, d), 91).view(np.uint16).copy()
    V = synth.fp16_np((40, d), 92).view(np.uint16)
    q = synth.fp16_np((1, d), 93).view(np.uint16)
    K[17] = q[0]
    e = np.zeros((0, d), np.uint16)
    out = O.attention_regions(q, K, V, e, e, 10.0)
    np.testing.assert_allclose(out[0], O.fp16_to_f64(V[17]), rtol=1e-6, atol=1e-8)


def test_empty_cache_rejected():
    e = np.zeros((0, 128), np.uint16)
    with pytest.raises(ValueError):
        O.attention_regions(np.zeros((1, 128), np.uint16), e, e, e, e, 1.0)
