"""Pins of the prune-then-quantize payload oracle ("we first prune each
token's KV cache before quantization is performed", KIVI 4-bit of tab:joint_quant; SPEC S:486-503
quantize_group / prune_then_quantize). Readings R25-R27: asymmetric 4-bit per-token
groups over the kept values, float32 quantizer arithmetic, one fp16 rounding on reconstruction."""
import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import synth
from oracle import mustafar_oracle as O


def f16(xs):
    return np.asarray(xs, np.float16).view(np.uint16)


def vals(bits):
    return np.asarray(bits, np.uint16).view(np.float16).astype(np.float64)


def test_constant_group_reconstructs_exactly():
    """a constant group (max = min) uses scale 1, every code is 0, reconstruction exact."""
    sc, z, q = O.quantize_group(f16([0.75] * 7))
    assert float(np.array(sc, np.uint16).view(np.float16)) == 1.0
    assert q.tolist() == [0] * 7
    assert np.array_equal(O.dequantize_group(sc, z, q), f16([0.75] * 7))


def test_integer_lattice_reconstructs_exactly():
    """4-bit codes on {0, 1, ..., 15}: min 0, scale 15/15 = 1, codes = values, exact."""
    x = f16(np.arange(16)[::-1])
    sc, z, q = O.quantize_group(x)
    assert q.tolist() == list(range(16))[::-1]
    assert np.array_equal(O.dequantize_group(sc, z, q), x)


def test_hand_example():
    """[1.0, 2.5, -0.5, 4.0]: zero = -0.5, span = 4.5, scale = f16(4.5 / 15 = 0.3) = 0x34CD =
    1.2001953125 * 2^-2 = 0.300048828125; codes rint((x + 0.5) / 0.300048828125) =
    rint([4.9992, 9.9984, 0, 14.9976]) = [5, 10, 0, 15]; reconstruction 5 * s - 0.5 =
    1.000244140625 -> f16 1.0 (spacing 2^-10), 10 * s - 0.5 = 2.50048828125 -> 2.5 (2^-9),
    15 * s - 0.5 = 4.000732421875 -> 4.0 (2^-8)."""
    sc, z, q = O.quantize_group(f16([1.0, 2.5, -0.5, 4.0]))
    assert sc == 0x34CD and z == f16([-0.5])[0]
    assert q.tolist() == [5, 10, 0, 15]
    assert vals(O.dequantize_group(sc, z, q)).tolist() == [1.0, 2.5, -0.5, 4.0]


def test_half_step_rounds_to_even():
    """Round half to even: values {0, 1, 1.5, ..., } with span 15 put x = 1.5 exactly half
    way between codes 1 and 2 -> 2; x = 2.5 -> 2; x = 3.5 -> 4."""
    sc, z, q = O.quantize_group(f16([0.0, 15.0, 1.5, 2.5, 3.5]))
    assert float(np.array(sc, np.uint16).view(np.float16)) == 1.0
    assert q.tolist() == [0, 15, 2, 2, 4]


@settings(max_examples=300, deadline=None)
@given(st.lists(st.floats(min_value=-300, max_value=300, allow_nan=False, width=16), min_size=1, max_size=64))
def test_error_bound_and_idempotence(xs):
    """Reconstruction error per kept value <= (1/2 + 1e-5) * scale + half an fp16 ulp of the result
    (S:490 bound; the float32 quantizer moves r by < 1e-5 and the fp16 rounding of code * scale +
    zero adds half an ulp); re-quantizing the reconstruction reproduces the codes."""
    x = f16(xs)
    sc, z, q = O.quantize_group(x)
    xh = O.dequantize_group(sc, z, q)
    s = float(np.array(sc, np.uint16).view(np.float16))
    err = np.abs(vals(xh) - vals(x))
    assert np.all(err <= 0.5 * s * (1 + 1e-5) + np.abs(vals(xh)) * 2.0 ** -11 + 1e-12)
    assert np.all(q <= 15)
    sc2, z2, q2 = O.quantize_group(xh)
    assert np.array_equal(q, q2)


def test_records_round_trip_and_layout():
    """prune_then_quantize: the selection is the magnitude top-k (unchanged bitmap and
    offsets), pruned entries reconstruct to exact zero, kept entries within the bound, record bytes
    laid out as R26 (scale, zero, nibbles low-first, zero padding)."""
    T, d, k = 50, 128, 39
    bits = synth.fp16_np((T, d), 321).view(np.uint16)
    keep = O.prune_tokens(bits, k)
    bm, rec, off = O.compress_tokens_q4(bits, keep, k)
    bm16, vals16, off16 = O.compress_tokens(bits, keep, k)
    assert np.array_equal(bm, bm16) and np.array_equal(off, off16)
    assert rec.shape == (T, O.q4_record_bytes(k)) == (T, 32)
    dense = O.decompress_tokens_q4(bm, rec, off, k, d)
    assert np.all(dense[~keep] == 0)
    for t in range(T):
        sc, z, q = O.quantize_group(vals16[t, :k])
        assert rec[t, 0:2].view(np.uint16)[0] == sc and rec[t, 2:4].view(np.uint16)[0] == z
        nib = [(rec[t, 4 + i // 2] >> (4 * (i & 1))) & 0xF for i in range(k)]
        assert nib == q.tolist()
        assert np.array_equal(dense[t, keep[t]], O.dequantize_group(sc, z, q))
    assert np.all(rec[:, 4 + (k + 1) // 2:] == 0) and np.all(rec[:, 4 + k // 2] >> 4 == 0)


def test_all_keep_is_plain_group_quantization():
    """an all-keep mask reduces to plain quantization of the whole token vector."""
    bits = synth.fp16_np((3, 128), 9).view(np.uint16)
    keep = np.ones_like(bits, dtype=bool)
    bm, rec, off = O.compress_tokens_q4(bits, keep, 128)
    dense = O.decompress_tokens_q4(bm, rec, off, 128, 128)
    for t in range(3):
        sc, z, q = O.quantize_group(bits[t])
        assert np.array_equal(dense[t], O.dequantize_group(sc, z, q))


def test_corrupt_record_rejected():
    bits = synth.fp16_np((2, 128), 5).view(np.uint16)
    keep = O.prune_tokens(bits, 39)
    bm, rec, off = O.compress_tokens_q4(bits, keep, 39)
    bad = rec.copy()
    bad[0, -1] = 1
    with pytest.raises(O.FormatError):
        O.decompress_tokens_q4(bm, bad, off, 39, 128)
    bad = rec.copy()
    bad[1, 4 + 39 // 2] |= 0x30   # the unused high nibble of the last code byte
    with pytest.raises(O.FormatError):
        O.decompress_tokens_q4(bm, bad, off, 39, 128)


def test_cache_q4_attention_equals_dense_attention_on_reconstruction():
    """Alg. 1 over the quantized cache is plain attention over the reconstructed (dequantized,
    zero-filled) compressed tokens plus the exact window (the equivalence S:440 extended to the
    payload); prefill + appends equals a longer prefill record for record."""
    U, T, n, d, W = 2, 100, 40, 128, 32
    K = synth.fp16_np((U, T + n, d), 61).view(np.uint16)
    V = synth.fp16_np((U, T + n, d), 62).view(np.uint16)
    q = synth.fp16_np((U, 4, d), 63).view(np.uint16)
    c = O.OracleCache(U, d, 39, 39, W, T + n, value_bits=4)
    c.prefill(K[:, :T], V[:, :T])
    for i in range(n):
        c.append(K[:, T + i], V[:, T + i])
    c2 = O.OracleCache(U, d, 39, 39, W, T + n, value_bits=4)
    c2.prefill(K, V)
    for name in ("bitmap_k", "values_k", "offsets_k", "bitmap_v", "values_v", "offsets_v", "n_comp", "n_win"):
        assert np.array_equal(getattr(c, name), getattr(c2, name)), name
    out = O.attention(c, q, 0.125)
    for u in range(U):
        kc, vc, kl, vl = c.tokens(u)
        ref = O.attention_dense(q[u], np.concatenate([kc, kl]), np.concatenate([vc, vl]), 0.125)
        np.testing.assert_allclose(out[u], ref, rtol=1e-12, atol=1e-14)
