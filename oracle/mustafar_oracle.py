"""CPU oracle for the Mustafar hot path (arXiv 2505.22913).

TEST INFRASTRUCTURE ONLY. Nothing on the product path may import this module:
only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may call it. It shares no code with paper_2505_22913_b200/ (the CUDA path) and
imports nothing from it.

Plain, slow, obviously correct numpy in float64. Each function cites the passage it
follows: `P:n` = /root/reference/PAPER.md line n, `S:n` = SPEC.md line n. Where the
paper is silent the reading taken is the one listed in DESIGN.md "Readings" (R1..R17,
numbered as in SURVEY.md 8(c)).

What it computes:
  * keep_count          k = d - floor(s*d)                         (R1)
  * prune_tokens        per-token magnitude top-k, lower index pruned first on ties
                        (P:62 per-token pruning of K, P:173/P:178 of V; R2, R3)
  * compress_tokens     per-token bitmap records: 64-bit bitmap per 1x64 tile, packed
                        fp16 kept values in channel order padded with 0x0000 to a
                        multiple of 8, u32 tile offsets (R4-R8)
  * decompress_tokens   bitmap + values -> dense fp16 bits, validating the record
  * OracleCache         dense local window of W tokens + compressed history,
                        prefill-then-compress and evict-on-exit (R9, R12)
  * attention           Algorithm 1 in float64: scores over the compressed
                        and window tokens, one softmax over the concatenation, P.V (R10, R11)
  * size_model_paper    byte accounting of the paper's format orientation
  * query_abs_sum       output-aware accumulator w = sum over the window's queries and the
                        GQA group of |Q| (R21), float32 in a fixed order
  * attention_partial,  sequence split across ranks: one shard's softmax
    merge_partials      partials and their flash-decoding merge
  * key_scores,         per-token output-aware Key pruning: S = |K| * broadcast(w), top-k of
    prune_tokens_scored S per token, lower index pruned first on ties (R20)
  * quantize_group,     prune-then-quantize payload ("we first prune each
    dequantize_group,   token's KV cache before quantization is performed", KIVI 4-bit of
    compress_tokens_q4  tab:joint_quant): a token's kept values as 4-bit codes with an
                        asymmetric per-token fp16 scale / zero point (R25-R27)

Pins (tests/test_oracle*.py, `-m "not gpu"`): closed forms, the SPEC worked examples,
brute-force rank counting and exhaustive subsets on tiny inputs, the lossless round
trip, reduction to torch SDPA at sparsity 0, single-token / zero-query / permutation /
needle special cases, and the paper's compression ratios. No function here is
"parity unpinned".
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "keep_count", "k_pad_of", "magnitude", "prune_tokens", "apply_keep",
    "compress_tokens", "decompress_tokens", "FormatError", "OracleCache",
    "attention", "attention_dense", "size_model_paper", "size_model_build",
    "query_abs_sum", "key_scores", "prune_tokens_scored", "attention_partial", "merge_partials",
    "q4_record_bytes", "quantize_group", "dequantize_group", "compress_tokens_q4", "decompress_tokens_q4",
]


class FormatError(ValueError):
    """A compressed record violates the format invariants."""


# --------------------------------------------------------------------------- pruning
def keep_count(sparsity: float, d: int) -> int:
    """Kept channels per token: k = d - floor(s*d) (R1; S:115 'p = floor(s x cols)')."""
    if not (0.0 <= sparsity < 1.0):
        raise ValueError("sparsity must be in [0,1)")
    return int(d - math.floor(sparsity * d))


def k_pad_of(k: int) -> int:
    """Packed-value slots per token: k rounded up to a multiple of 8 (P:441 'multiples-of-8
    padding'; R7 pads per token)."""
    return ((k + 7) // 8) * 8


def magnitude(bits: np.ndarray) -> np.ndarray:
    """|x| of an fp16 bit pattern as an unsigned integer: bits & 0x7FFF (R3). Orders finite
    fp16 magnitudes exactly, subnormals included; +0 and -0 compare equal."""
    return (np.asarray(bits, dtype=np.uint16) & np.uint16(0x7FFF)).astype(np.int64)


def prune_tokens(bits: np.ndarray, k: int) -> np.ndarray:
    """Per-token magnitude pruning (P:62, P:173, P:178 'per-token magnitude-based pruning').

    bits: uint16 [..., d] fp16 bit patterns, one token vector per row.
    Returns bool keep mask [..., d] with exactly k True per row.

    Plain definition: stable-sort each row's channels by (magnitude ascending, channel
    index ascending) and prune the first d-k (R2: 'ties broken by pruning the lower
    channel index first')."""
    bits = np.asarray(bits, dtype=np.uint16)
    d = bits.shape[-1]
    if not (1 <= k <= d):
        raise ValueError("k must be in [1, d]")
    mag = magnitude(bits)
    idx = np.broadcast_to(np.arange(d, dtype=np.int64), mag.shape)
    order = np.lexsort((idx, mag), axis=-1)          # primary key mag, secondary idx
    keep = np.ones(bits.shape, dtype=bool)
    pruned = order[..., : d - k]
    np.put_along_axis(keep, pruned, False, axis=-1)
    return keep


def query_abs_sum(q_ring: np.ndarray) -> np.ndarray:
    """Output-aware accumulator (P:86 'the element-wise L1 accumulation of the current and
    next 31 Query vector'; P:93 'For GQA ... we sum the pruning score of all queries mapped
    to each KV cache').

    q_ring: uint16 fp16 bit patterns [U, R, G, d]: the R queries of the window (slot order) of
    each unit's G query heads. Returns float32 [U, d]: w[u, c] = sum_r sum_g |q[u, r, g, c]|.

    R21: float32, added one term at a time in the order r ascending, then g ascending (the
    kernel's precision and order, so both sides hold the same bits)."""
    q = np.asarray(q_ring, dtype=np.uint16)
    U, R, G, d = q.shape
    a = np.abs(q.view(np.float16).astype(np.float32))
    w = np.zeros((U, d), dtype=np.float32)
    for r in range(R):
        for g in range(G):
            w = (w + a[:, r, g, :]).astype(np.float32)   # one float32 add per term
    return w


def key_scores(bits: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Per-token output-aware Key score S = |K| (.) broadcast(w). bits: uint16 [..., d]
    fp16 token vectors; w: float32 [d] (or broadcastable), finite and >= 0.

    R20: |K| is the fp16 magnitude widened exactly to float32; the product is one float32
    multiply, rounded to nearest (the kernel's precision)."""
    k = np.abs(np.asarray(bits, dtype=np.uint16).view(np.float16).astype(np.float32))
    return (k * np.asarray(w, dtype=np.float32)).astype(np.float32)


def prune_tokens_scored(scores: np.ndarray, k: int) -> np.ndarray:
    """Keep the k largest scores per row (P:91 'The absolute value of the score element ...
    is used to decide the elements to be pruned within a token's Key vector'); scores are
    >= 0, so |S| = S. Ties: the lower channel index is pruned first (R2), as in prune_tokens.
    Returns bool keep mask with exactly k True per row."""
    sc = np.asarray(scores, dtype=np.float32)
    d = sc.shape[-1]
    if not (1 <= k <= d):
        raise ValueError("k must be in [1, d]")
    if np.isnan(sc).any() or (sc < 0).any():
        raise ValueError("scores must be >= 0")
    idx = np.broadcast_to(np.arange(d, dtype=np.int64), sc.shape)
    order = np.lexsort((idx, sc.astype(np.float64)), axis=-1)
    keep = np.ones(sc.shape, dtype=bool)
    np.put_along_axis(keep, order[..., : d - k], False, axis=-1)
    return keep


def apply_keep(bits: np.ndarray, keep: np.ndarray) -> np.ndarray:
    """Pruned entries become 0x0000; kept entries are copied bit-for-bit."""
    return np.where(keep, np.asarray(bits, dtype=np.uint16), np.uint16(0)).astype(np.uint16)


# --------------------------------------------------------------------------- format
def compress_tokens(bits: np.ndarray, keep: np.ndarray, k: int, first_record: int = 0):
    """Bitmap-based sparse format (P:218 'compressed tiles corresponding to a 1x64 column ...
    Per-tile bitmap of 64 bits ... tile offset is used to address the correct position of
    each tile's starting non-zero'; P:441 'multiples-of-8 padding').

    Build layout (R4-R8): one record per token vector,
      bitmap  u64 [T, d/64]   bit i of tile j  <=> channel 64j+i kept (LSB first)
      values  u16 [T, k_pad]  kept fp16 bit patterns in ascending channel order, then 0x0000
      offsets u32 [T, d/64]   (first_record+t)*k_pad + number of kept channels in tiles < j
    """
    bits = np.asarray(bits, dtype=np.uint16)
    keep = np.asarray(keep, dtype=bool)
    T, d = bits.shape
    assert d % 64 == 0
    kp = k_pad_of(k)
    nt = d // 64
    if T and not np.all(keep.sum(axis=1) == k):
        raise ValueError("every token must keep exactly k channels")
    bm = np.packbits(keep.reshape(T, nt, 64), axis=-1, bitorder="little")   # [T, nt, 8] bytes
    bitmap = bm.reshape(T, nt * 8).copy().view("<u8").reshape(T, nt)
    values = np.zeros((T, kp), dtype=np.uint16)
    if T:
        values[:, :k] = bits[keep].reshape(T, k)   # row-major boolean gather = channel order
    per_tile = keep.reshape(T, nt, 64).sum(axis=2)
    before = np.concatenate([np.zeros((T, 1), np.int64), np.cumsum(per_tile, axis=1)[:, :-1]], axis=1)
    rec = np.arange(first_record, first_record + T, dtype=np.int64)[:, None]
    offsets = (rec * kp + before).astype(np.uint32)
    return bitmap.astype(np.uint64), values, offsets


def decompress_tokens(bitmap: np.ndarray, values: np.ndarray, offsets: np.ndarray | None,
                      k: int, d: int, first_record: int = 0) -> np.ndarray:
    """Inverse of compress_tokens (the paper's 'extract' step), with validation:
    popcount == k per token (R4), padding slots are 0x0000 (R7), offsets equal the
    prefix popcounts (R8). Raises FormatError on any violation."""
    bitmap = np.asarray(bitmap, dtype=np.uint64)
    values = np.asarray(values, dtype=np.uint16)
    T, nt = bitmap.shape
    assert nt * 64 == d
    kp = k_pad_of(k)
    if values.shape != (T, kp):
        raise FormatError("values shape")
    keep = np.unpackbits(bitmap.view(np.uint8).reshape(T, nt * 8), axis=-1,
                         bitorder="little").astype(bool)
    if T and not np.all(keep.sum(axis=1) == k):
        raise FormatError("bitmap popcount != k")
    if T and np.any(values[:, k:] != 0):
        raise FormatError("non-zero padding")
    if offsets is not None:
        per_tile = keep.reshape(T, nt, 64).sum(axis=2)
        before = np.concatenate([np.zeros((T, 1), np.int64), np.cumsum(per_tile, axis=1)[:, :-1]], axis=1)
        rec = np.arange(first_record, first_record + T, dtype=np.int64)[:, None]
        if not np.array_equal(np.asarray(offsets, dtype=np.int64), rec * kp + before):
            raise FormatError("tile offsets inconsistent with bitmaps")
    out = np.zeros((T, d), dtype=np.uint16)
    if T:
        out[keep] = values[:, :k].reshape(-1)
    return out


# --------------------------------------------------------------------------- 4-bit payload
def q4_record_bytes(k: int) -> int:
    """Bytes of one token's quantized payload (R26): fp16 scale, fp16 zero point, ceil(k/2) bytes
    of 4-bit codes, zero-padded to a multiple of 16 bytes (16-byte aligned records, as R7)."""
    return ((4 + (k + 1) // 2 + 15) // 16) * 16


def quantize_group(vals: np.ndarray):
    """S:489-490 quantize_group with bits = 4 (KIVI 4-bit; tab:joint_quant): asymmetric
    uniform mapping, q_max = 15, zero point = min, scale = (max - min) / q_max (1 when that is 0),
    round half to even. R25 fixes the arithmetic (float32, the kernel's precision, like R20):
        span  = f32(max) - f32(min)            scale = f16(span / 15), 1.0 if 0 or not finite
        inv   = 1 / f32(scale)                 code  = rint(min(max((f32(x) - f32(zero)) * inv, 0), 15))
    every operation rounded to nearest in float32 (rint: half to even); max(NaN, 0) = 0.
    vals: uint16 fp16 bits [n >= 1] (a token's kept values). Returns (scale bits, zero bits,
    codes uint8 [n])."""
    b = np.asarray(vals, dtype=np.uint16)
    if b.size == 0:
        raise ValueError("empty group")
    if not np.all(np.isfinite(b.view(np.float16))):
        raise ValueError("non-finite input (S:491)")
    v = b.view(np.float16)
    # min / max in the total order of fp16 values with -0 < +0 (R25: the zero point's sign is
    # well defined when both zeros are kept): order key = bits ^ 0x8000 for x >= +0, ~bits else
    key = np.where(b & 0x8000, (~b) & 0xFFFF, b | 0x8000).astype(np.int64)
    lo, hi = v[np.argmin(key)], v[np.argmax(key)]
    span = np.float32(hi) - np.float32(lo)
    sc = np.float16(np.float32(span) / np.float32(15.0))
    if not np.isfinite(sc) or sc == 0:
        sc = np.float16(1.0)
    inv = np.float32(1.0) / np.float32(sc)
    with np.errstate(invalid="ignore", over="ignore"):
        r = (v.astype(np.float32) - np.float32(lo)) * inv
        q = np.rint(np.fmin(np.fmax(r, np.float32(0)), np.float32(15)))
    return (np.array(sc, np.float16).view(np.uint16).item(), np.array(lo, np.float16).view(np.uint16).item(),
            q.astype(np.uint8))


def dequantize_group(scale_bits: int, zero_bits: int, codes: np.ndarray) -> np.ndarray:
    """Inverse map: x = f16(code * scale + zero), the exact value rounded once to fp16 (a
    correctly rounded fp16 fused multiply-add). Returns uint16 fp16 bits."""
    sc = float(np.array(scale_bits, np.uint16).view(np.float16))
    z = float(np.array(zero_bits, np.uint16).view(np.float16))
    exact = np.asarray(codes, dtype=np.float64) * sc + z        # exact in float64 (15 x 11-bit products)
    return exact.astype(np.float16).view(np.uint16)


def compress_tokens_q4(bits: np.ndarray, keep: np.ndarray, k: int, first_record: int = 0):
    """Bitmap format with the prune-then-quantize payload: bitmaps and tile
    offsets exactly as compress_tokens (the selection is unchanged: prune first), and per
    token one record of q4_record_bytes(k) bytes:
      [0:2] scale fp16, [2:4] zero fp16, [4 + i//2] code of kept value i (channel order; low nibble
      for even i), remaining bytes 0x00.
    Returns (bitmap u64 [T, d/64], records u8 [T, RQ], offsets u32 [T, d/64])."""
    bits = np.asarray(bits, dtype=np.uint16)
    keep = np.asarray(keep, dtype=bool)
    bitmap, values, offsets = compress_tokens(bits, keep, k, first_record)
    T = bits.shape[0]
    rq = q4_record_bytes(k)
    rec = np.zeros((T, rq), dtype=np.uint8)
    for t in range(T):
        sc, z, q = quantize_group(values[t, :k])
        rec[t, 0:2] = np.array([sc], np.uint16).view(np.uint8)
        rec[t, 2:4] = np.array([z], np.uint16).view(np.uint8)
        for i, c in enumerate(q):
            rec[t, 4 + i // 2] |= np.uint8(int(c) << (4 * (i & 1)))
    return bitmap, rec, offsets


def decompress_tokens_q4(bitmap, records, offsets, k: int, d: int, first_record: int = 0) -> np.ndarray:
    """Dense fp16 bits [T, d] of quantized records: dequantized kept values at the bitmap's
    positions, exact zeros at pruned channels ("pruned entries remain exact zero"), with
    validation of the bitmap (popcount k), the offsets, and the record's zero padding."""
    bitmap = np.asarray(bitmap, dtype=np.uint64)
    records = np.asarray(records, dtype=np.uint8)
    T, nt = bitmap.shape
    rq = q4_record_bytes(k)
    if records.shape != (T, rq):
        raise FormatError("record shape")
    used = 4 + (k + 1) // 2
    if T and np.any(records[:, used:] != 0):
        raise FormatError("non-zero record padding")
    if T and k % 2 and np.any(records[:, 4 + k // 2] >> 4):
        raise FormatError("non-zero unused nibble")
    zeros_vals = np.zeros((T, k_pad_of(k)), np.uint16)   # validate bitmaps / offsets only
    decompress_tokens(bitmap, zeros_vals, offsets, k, d, first_record)
    keep = np.unpackbits(bitmap.view(np.uint8).reshape(T, nt * 8), axis=-1, bitorder="little").astype(bool)
    out = np.zeros((T, d), dtype=np.uint16)
    for t in range(T):
        sc = int(records[t, 0:2].view(np.uint16)[0])
        z = int(records[t, 2:4].view(np.uint16)[0])
        codes = np.array([(records[t, 4 + i // 2] >> (4 * (i & 1))) & 0xF for i in range(k)], np.uint8)
        out[t, keep[t]] = dequantize_group(sc, z, codes)
    return out


def fp16_to_f64(bits: np.ndarray) -> np.ndarray:
    """Exact fp16 -> float64 (every fp16 value is representable in float64)."""
    return np.asarray(bits, dtype=np.uint16).view(np.float16).astype(np.float64)


# --------------------------------------------------------------------------- cache
class OracleCache:
    """KV cache semantics of P:58 ('the recent 32 tokens remain untouched') and P:234
    ('KV cache generated in prefill stage is pruned and compressed before the start of
    decode stage ... KV cache generated in decode stage is kept as-is (dense) while it is
    within the local window, then pruned and compressed afterwards').

    Readings: R9 (the last min(T, W) prefill tokens stay dense; decode tokens are evicted
    one at a time as they leave the window), R12 (append precedes attention).

    State, per unit u (a (batch, kv-head) pair; U = B * Hkv, b-major), mirroring the
    device buffers of include/mustafar.h so they can be compared byte for byte:
      bitmap_k/v [U][cap][d/64] u64, values_k/v [U][cap][k_pad] u16,
      offsets_k/v [U][cap][d/64] u32, win_k/v [U][W][d] u16 (token p in slot p % W),
      n_comp [U], n_win [U].
    Token p of unit u is compressed into record p (records are in chronological order).
    """

    def __init__(self, U: int, d: int, keep_k: int, keep_v: int, window: int, capacity: int,
                 value_bits: int = 16):
        self.U, self.d, self.kk, self.kv, self.W, self.cap = U, d, keep_k, keep_v, window, capacity
        if value_bits not in (16, 4):
            raise ValueError("value_bits must be 16 or 4")
        self.value_bits = value_bits   # 4: prune-then-quantize payload
        self.nt = d // 64
        self.kpk, self.kpv = k_pad_of(keep_k), k_pad_of(keep_v)
        z = np.zeros
        self.bitmap_k = z((U, capacity, self.nt), np.uint64)
        self.bitmap_v = z((U, capacity, self.nt), np.uint64)
        if value_bits == 16:
            self.values_k = z((U, capacity, self.kpk), np.uint16)
            self.values_v = z((U, capacity, self.kpv), np.uint16)
        else:   # quantized records [U][cap][q4_record_bytes(k)] bytes
            self.values_k = z((U, capacity, q4_record_bytes(keep_k)), np.uint8)
            self.values_v = z((U, capacity, q4_record_bytes(keep_v)), np.uint8)
        self.offsets_k = z((U, capacity, self.nt), np.uint32)
        self.offsets_v = z((U, capacity, self.nt), np.uint32)
        self.win_k = z((U, max(window, 1), d), np.uint16)
        self.win_v = z((U, max(window, 1), d), np.uint16)
        self.n_comp = z(U, np.int64)
        self.n_win = z(U, np.int64)
        self.key_weights = None   # float32 [U, d]: output-aware K pruning when set

    def set_key_weights(self, w):
        """Output-aware K pruning for every later K compression (prefill and evictions) with
        S = |K| * w[u] (key_scores); None restores magnitude pruning. V is always pruned by
        magnitude (per-token magnitude is already output-aware for V)."""
        self.key_weights = None if w is None else np.asarray(w, dtype=np.float32).copy()

    # -- one tensor, one unit: compress tokens (given as bits) into records r0..r0+T-1
    def _store(self, which: str, u: int, r0: int, bits: np.ndarray):
        k = self.kk if which == "k" else self.kv
        if r0 + bits.shape[0] > self.cap:
            raise OverflowError("compressed capacity exceeded")
        if which == "k" and self.key_weights is not None:
            keep = prune_tokens_scored(key_scores(bits, self.key_weights[u]), k)
        else:
            keep = prune_tokens(bits, k)
        if self.value_bits == 16:
            bm, vals, offs = compress_tokens(bits, keep, k, first_record=r0)
        else:
            bm, vals, offs = compress_tokens_q4(bits, keep, k, first_record=r0)
        getattr(self, "bitmap_" + which)[u, r0:r0 + len(bits)] = bm
        getattr(self, "values_" + which)[u, r0:r0 + len(bits)] = vals
        getattr(self, "offsets_" + which)[u, r0:r0 + len(bits)] = offs

    def prefill(self, K: np.ndarray, V: np.ndarray, lengths=None):
        """K, V: uint16 [U, T, d]. Unit u ingests its first lengths[u] tokens (default T)."""
        U, T, d = K.shape
        assert U == self.U and d == self.d
        lengths = [T] * U if lengths is None else list(lengths)
        for u in range(U):
            L = int(lengths[u])
            nd = min(L, self.W)
            nc = L - nd
            self._store("k", u, 0, K[u, :nc])
            self._store("v", u, 0, V[u, :nc])
            self.win_k[u].fill(0)
            self.win_v[u].fill(0)
            for p in range(nc, L):
                self.win_k[u, p % self.W] = K[u, p]
                self.win_v[u, p % self.W] = V[u, p]
            self.n_comp[u], self.n_win[u] = nc, nd

    def append(self, k_new: np.ndarray, v_new: np.ndarray):
        """k_new, v_new: uint16 [U, d]; one decode token per unit."""
        for u in range(self.U):
            nc, nw = int(self.n_comp[u]), int(self.n_win[u])
            if self.W == 0:
                self._store("k", u, nc, k_new[u][None])
                self._store("v", u, nc, v_new[u][None])
                self.n_comp[u] = nc + 1
                continue
            if nw == self.W:                        # oldest window token exits the window
                slot = nc % self.W
                self._store("k", u, nc, self.win_k[u, slot][None].copy())
                self._store("v", u, nc, self.win_v[u, slot][None].copy())
                nc += 1
                nw -= 1
            p = nc + nw                             # chronological position of the new token
            self.win_k[u, p % self.W] = k_new[u]
            self.win_v[u, p % self.W] = v_new[u]
            self.n_comp[u], self.n_win[u] = nc, nw + 1

    def tokens(self, u: int):
        """Decompressed K, V of unit u in chronological order (compressed first, then the
        window), as fp16 bit patterns [n, d] -- Alg. 1's K_C, V_C then K_L, V_L."""
        nc, nw = int(self.n_comp[u]), int(self.n_win[u])
        dec = decompress_tokens if self.value_bits == 16 else decompress_tokens_q4
        kc = dec(self.bitmap_k[u, :nc], self.values_k[u, :nc], self.offsets_k[u, :nc], self.kk, self.d)
        vc = dec(self.bitmap_v[u, :nc], self.values_v[u, :nc], self.offsets_v[u, :nc], self.kv, self.d)
        slots = [(nc + i) % max(self.W, 1) for i in range(nw)]
        kl = self.win_k[u, slots] if nw else np.zeros((0, self.d), np.uint16)
        vl = self.win_v[u, slots] if nw else np.zeros((0, self.d), np.uint16)
        return kc, vc, kl, vl


# --------------------------------------------------------------------------- attention
def attention(cache: OracleCache, q: np.ndarray, scale: float, units=None) -> np.ndarray:
    """Algorithm 1, float64, for every unit and each of its G query heads.

    q: fp16 bits [U, G, d] (== [B, Hq, d] with h_kv = floor(h_q / G), R11).
      S_L = scale * Q_t K_L ; S_C = scale * Q_t K_C          (lines 1-2; scale: R10)
      S_t = softmax(concat(S_C, S_L))                          (line 3)
      O_t = V_C S_C^T + V_L S_L^T                              (lines 4-5)
    Returns float64 [len(units), G, d]."""
    units = range(cache.U) if units is None else units
    out = []
    for u in units:
        kc, vc, kl, vl = cache.tokens(u)
        out.append(attention_regions(q[u], kc, vc, kl, vl, scale))
    return np.stack(out) if out else np.zeros((0,) + q.shape[1:], np.float64)


def attention_regions(qu, kc, vc, kl, vl, scale):
    """Alg. 1 for one unit: qu [G, d] fp16 bits; K_C/V_C, K_L/V_L fp16 bits [n, d]."""
    Q = fp16_to_f64(qu)
    KC, VC, KL, VL = (fp16_to_f64(x) for x in (kc, vc, kl, vl))
    if KC.shape[0] + KL.shape[0] == 0:
        raise ValueError("attention over an empty cache")
    s_c = scale * (Q @ KC.T)                       # line 2
    s_l = scale * (Q @ KL.T)                       # line 1
    s = np.concatenate([s_c, s_l], axis=1)         # concat(S_C, S_L)
    m = s.max(axis=1, keepdims=True)
    e = np.exp(s - m)
    p = e / e.sum(axis=1, keepdims=True)           # line 3 softmax
    p_c, p_l = p[:, : KC.shape[0]], p[:, KC.shape[0]:]   # line 4 split
    return p_c @ VC + p_l @ VL                     # line 5


def attention_partial(cache: OracleCache, q: np.ndarray, scale: float):
    """One shard's Algorithm 1 stopped before the normalisation of line 3: the
    softmax partials over this cache's tokens (flash-decoding state), float64,
    natural-log units:
      m = max_t s_t,  l = sum_t exp(s_t - m),  o = sum_t exp(s_t - m) v_t
    with s_t = scale * q . k_t over the compressed and window tokens (R10). Returns (m [U, G],
    l [U, G], o [U, G, d]); a unit without tokens gives m = -inf, l = 0, o = 0."""
    U, G, d = cache.U, q.shape[1], cache.d
    m = np.full((U, G), -np.inf)
    l = np.zeros((U, G))
    o = np.zeros((U, G, d))
    for u in range(U):
        kc, vc, kl, vl = cache.tokens(u)
        K = fp16_to_f64(np.concatenate([kc, kl], axis=0))
        V = fp16_to_f64(np.concatenate([vc, vl], axis=0))
        if K.shape[0] == 0:
            continue
        s = scale * (fp16_to_f64(q[u]) @ K.T)
        m[u] = s.max(axis=1)
        e = np.exp(s - m[u][:, None])
        l[u] = e.sum(axis=1)
        o[u] = e @ V
    return m, l, o


def merge_partials(parts):
    """Merge shards' partials [(m, l, o), ...] into O (the a9 split combine; natural units):
    M = max_i m_i, O = sum_i exp(m_i - M) o_i / sum_i exp(m_i - M) l_i. Shards with m = -inf
    contribute nothing."""
    M = np.max(np.stack([p[0] for p in parts]), axis=0)
    num = np.zeros_like(parts[0][2])
    den = np.zeros_like(parts[0][1])
    for m, l, o in parts:
        w = np.where(np.isneginf(m), 0.0, np.exp(np.where(np.isneginf(m), 0.0, m - M)))
        num += w[..., None] * o
        den += w * l
    return num / den[..., None]


def attention_dense(q: np.ndarray, K: np.ndarray, V: np.ndarray, scale: float) -> np.ndarray:
    """Textbook softmax(scale * q K^T) V in float64 over fp16-bit inputs; q [G, d], K/V [n, d].
    The dense-KV reference the sparse path reduces to when nothing is pruned."""
    Q, Kd, Vd = fp16_to_f64(q), fp16_to_f64(K), fp16_to_f64(V)
    s = scale * (Q @ Kd.T)
    e = np.exp(s - s.max(axis=1, keepdims=True))
    return (e / e.sum(axis=1, keepdims=True)) @ Vd


# --------------------------------------------------------------------------- byte accounting
def _pad8(n):
    return ((np.asarray(n) + 7) // 8) * 8


def size_model_paper(keep_k, keep_v, W: int = 32, group: int = 64, elem: int = 2,
                     bitmap_bytes: int = 8, offset_bytes: int = 4):
    """Bytes of one head's cache in the paper's orientation (S:223-226,
    S:247-259): K tiles are 64 tokens x 1 channel, V tiles 1 token x 64 channels; every tile
    costs bitmap + offset + pad8(nnz) * elem; tokens not in a full 64-token group (the dense
    local window and the group tail) stay dense. keep_k / keep_v: bool [T, d] or None (dense).
    Returns (compressed_bytes, dense_bytes)."""
    ref = keep_k if keep_k is not None else keep_v
    T, d = ref.shape
    ncomp = ((max(T - W, 0)) // group) * group
    total = 0
    for keep, kind in ((keep_k, "k"), (keep_v, "v")):
        if keep is None:
            total += T * d * elem
            continue
        body = keep[:ncomp]
        if kind == "k":   # column tiling across the token dimension
            nnz = body.reshape(ncomp // group, group, d).sum(axis=1).reshape(-1)
        else:             # column tiling across the channel dimension
            nnz = body.reshape(ncomp, d // 64, 64).sum(axis=2).reshape(-1)
        total += int(np.sum(_pad8(nnz) * elem + bitmap_bytes + offset_bytes))
        total += (T - ncomp) * d * elem
    return total, 2 * T * d * elem


def size_model_build(T: int, d: int, keep_k: int | None, keep_v: int | None, W: int = 32,
                     with_offsets: bool = True):
    """Bytes of one head's cache in the build's per-token record layout (R5-R8): per
    compressed token and tensor d/64 * 8 B bitmap + 2*k_pad B values (+ d/64 * 4 B offsets);
    the last min(T, W) tokens dense. Returns (compressed_bytes, dense_bytes)."""
    nd = min(T, W)
    nc = T - nd
    total = 0
    for k in (keep_k, keep_v):
        if k is None:
            total += T * d * 2
            continue
        rec = (d // 64) * 8 + 2 * k_pad_of(k) + ((d // 64) * 4 if with_offsets else 0)
        total += nc * rec + nd * d * 2
    return total, 2 * T * d * 2
