// compress_dev.cuh -- device code of K1 (per-token magnitude pruning + bitmap compression)
// shared by compress.cu (prefill / append kernels) and attn_warp.cu (fused decode step).
// See compress.cu for the method and its citations.
#pragma once
#include <cstdint>

#include "kernels.cuh"
#include "ptx.cuh"

namespace mstf {

// Warp-wide u32 reductions as inline PTX: every caller reaches them with the whole warp
// converged (warp-uniform control flow), and the intrinsics' divergence-safe lowering
// (WARPSYNC.COLLECTIVE around each REDUX) cost the old prefill kernel most of its time.
__device__ __forceinline__ uint32_t warp_sum(uint32_t x) {
  uint32_t r;
  asm volatile("redux.sync.add.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(x));
  return r;
}
__device__ __forceinline__ uint32_t warp_or(uint32_t x) {
  uint32_t r;
  asm volatile("redux.sync.or.b32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(x));
  return r;
}

// Keep nibble for keys m[4] (lane l: channels 4l..4l+3) given tau = the k-th largest key:
// keys > tau are kept; among keys == tau the (k - #{key > tau}) highest channel indices (R2:
// the lower index is pruned first). Warp-uniform control flow.
__device__ __forceinline__ uint32_t keep_nibble_at(const uint32_t (&m)[4], uint32_t tau, uint32_t k) {
  uint32_t nib = 0, ge = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    nib |= (uint32_t)(m[j] >= tau) << j;
    ge += m[j] >= tau;
  }
  ge = warp_sum(ge);
  if (ge > k) {  // warp-uniform: ties at tau
    uint32_t gt = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) gt += m[j] > tau;
    const uint32_t need = k - warp_sum(gt);  // >= 1 slots for channels with key == tau
    const uint32_t gtm = lanemask_gt();
    uint32_t above = 0;
    bool eq[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      eq[j] = (m[j] == tau);
      above += __popc(__ballot_sync(0xffffffffu, eq[j]) & gtm);
    }
    nib = 0;
#pragma unroll
    for (int j = 3; j >= 0; --j) {
      const bool keep = (m[j] > tau) || (eq[j] && above < need);
      if (eq[j]) ++above;
      nib |= (uint32_t)keep << j;
    }
  }
  return nib;
}

// Top-k selection of one token vector (a1, a2): lane l holds channels 4l..4l+3 as raw fp16
// bits (x: channels 4l, 4l+1; y: 4l+2, 4l+3). Returns the lane's 4-bit keep nibble (bit j <->
// channel 4l+j). Exactly k bits are set over the warp.
//   tau = max t such that #{c : mag_c >= t} >= k, found MSB-first. SWAR compares: with the
//   top bit of each field set, (field | top) - cand keeps the top bit iff field >= cand and
//   never borrows across fields. Bits 14..8 compare the high bytes (4 per register), bits
//   7..0 the full 15-bit magnitudes (2 per register).
//   Ties at tau (only when #{mag >= tau} > k): keep the (k - #{mag > tau}) highest channel
//   indices among mag == tau (R2: the lower index is pruned first).
__device__ __forceinline__ uint32_t select_keep_nibble(uint32_t x, uint32_t y, uint32_t k, int lane) {
  const uint32_t mx = x & 0x7FFF7FFFu, my = y & 0x7FFF7FFFu;
  // phase 1: bits 14..8 on the high bytes of the four magnitudes. The lane's flags (top bit
  // of each byte) move to bit 0 of their bytes with a multiply-high and are summed into the
  // top byte with a multiply, both on the FMA pipe; the warp sum of that byte (<= 128; the
  // lower bytes never carry into it) is compared against k << 24.
  const uint32_t hb = __byte_perm(mx, my, 0x7531) | 0x80808080u;
  const uint32_t k24 = k << 24, k16 = k << 16;
  uint32_t t4 = 0;  // tau >> 8, replicated in 4 bytes
#pragma unroll
  for (int b = 6; b >= 0; --b) {
    const uint32_t c4 = t4 | (0x01010101u << b);
    const uint32_t f = __umulhi((hb - c4) & 0x80808080u, 1u << 25) * 0x01010101u;
    t4 = warp_sum(f) >= k24 ? c4 : t4;
  }
  // phase 2: bits 7..0 on the 15-bit magnitudes (flags at bits 0 and 16, summed into the
  // upper half)
  const uint32_t ax = mx | 0x80008000u, ay = my | 0x80008000u;
  uint32_t t2 = (t4 & 0x7Fu) * 0x01000100u;  // tau, replicated in 2 halves
#pragma unroll
  for (int b = 7; b >= 0; --b) {
    const uint32_t c2 = t2 | (0x00010001u << b);
    const uint32_t f = (__umulhi((ax - c2) & 0x80008000u, 1u << 17) + __umulhi((ay - c2) & 0x80008000u, 1u << 17)) *
                       0x00010001u;
    t2 = warp_sum(f) >= k16 ? c2 : t2;
  }
  const uint32_t tau = t2 & 0x7FFFu;
  const uint32_t m[4] = {mx & 0xFFFFu, mx >> 16, my & 0xFFFFu, my >> 16};
  return keep_nibble_at(m, tau, k);
}

// Output-aware variant (R20): keys are the float32 scores |x_c| * w_c (non-negative,
// so their bit patterns order like the values); tau by a 31-step MSB-first search.
__device__ __forceinline__ uint32_t select_keep_nibble_scored(uint32_t x, uint32_t y, float4 w, uint32_t k) {
  const uint32_t hv[4] = {x & 0x7FFFu, (x >> 16) & 0x7FFFu, y & 0x7FFFu, (y >> 16) & 0x7FFFu};
  const float wv[4] = {w.x, w.y, w.z, w.w};
  uint32_t m[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) m[j] = __float_as_uint(__fmul_rn(__half2float(__ushort_as_half((unsigned short)hv[j])), wv[j]));
  uint32_t tau = 0;
#pragma unroll 1
  for (int b = 30; b >= 0; --b) {
    const uint32_t cand = tau | (1u << b);
    const uint32_t n = warp_sum((uint32_t)(m[0] >= cand) + (uint32_t)(m[1] >= cand) + (uint32_t)(m[2] >= cand) +
                                (uint32_t)(m[3] >= cand));
    tau = n >= k ? cand : tau;
  }
  return keep_nibble_at(m, tau, k);
}

// Order key of an fp16 bit pattern: unsigned order == value order, with -0 < +0 (R25).
__device__ __forceinline__ uint32_t f16_order_key(uint32_t h) { return (h & 0x8000u) ? (~h & 0xFFFFu) : (h | 0x8000u); }
__device__ __forceinline__ uint32_t f16_from_key(uint32_t k) { return (k & 0x8000u) ? (k & 0x7FFFu) : (~k & 0xFFFFu); }
__device__ __forceinline__ uint32_t warp_min(uint32_t x) {
  uint32_t r;
  asm volatile("redux.sync.min.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(x));
  return r;
}
__device__ __forceinline__ uint32_t warp_max(uint32_t x) {
  uint32_t r;
  asm volatile("redux.sync.max.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(x));
  return r;
}

// 4-bit payload of one token: lane l holds the fp16 values h[4] of
// channels 4l..4l+3, keep nibble nib, and pos = kept channels of lower lanes. Writes the record
// [scale f16][zero f16][k nibbles, kept order, low nibble first][zero padding to rq bytes]:
// zero = least kept value (-0 < +0), scale = f16(f32(max - min) / 15) (1 if 0), code =
// rint(clamp((f32(x) - f32(zero)) * (1 / f32(scale)), 0, 15)), float32 round-to-nearest.
__device__ __forceinline__ void quantize_token_warp(const uint32_t (&h)[4], uint32_t nib, uint32_t pos, int k, int rq,
                                                    uint8_t* __restrict__ rec_out, int lane) {
  uint32_t kmin = 0xFFFFu, kmax = 0u;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t key = f16_order_key(h[j]);
    if (nib & (1u << j)) {
      kmin = min(kmin, key);
      kmax = max(kmax, key);
    }
  }
  kmin = warp_min(kmin);
  kmax = warp_max(kmax);
  const uint32_t zero_bits = f16_from_key(kmin), max_bits = f16_from_key(kmax);
  const float lo = __half2float(__ushort_as_half((unsigned short)zero_bits));
  const float hi = __half2float(__ushort_as_half((unsigned short)max_bits));
  __half sc = __float2half_rn(__fdiv_rn(__fsub_rn(hi, lo), 15.f));
  const float scf = __half2float(sc);
  if (!(scf != 0.f && isfinite(scf))) sc = __float2half_rn(1.f);
  const float inv = __frcp_rn(__half2float(sc));
  // this lane's codes in kept order as a nibble string, placed at nibble pos of the token
  uint32_t str = 0, n = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (nib & (1u << j)) {
      const float x = __half2float(__ushort_as_half((unsigned short)h[j]));
      const float r = fminf(fmaxf(__fmul_rn(__fsub_rn(x, lo), inv), 0.f), 15.f);
      str |= (uint32_t)rintf(r) << (4 * n);
      ++n;
    }
  }
  const unsigned long long placed = (unsigned long long)str << (4 * (pos & 7u));
  const uint32_t w0 = pos >> 3;
  const int ncw = (k + 7) >> 3;  // code words
  uint32_t mine = 0;             // record word lane (0: scale | zero, 1..: codes, rest: padding)
  for (int wi = 0; wi < ncw; ++wi) {
    const uint32_t part = (w0 == (uint32_t)wi ? (uint32_t)placed : 0u) | (w0 + 1 == (uint32_t)wi ? (uint32_t)(placed >> 32) : 0u);
    const uint32_t word = warp_or(part);
    if (lane == wi + 1) mine = word;
  }
  if (lane == 0) mine = (uint32_t)__half_as_ushort(sc) | (zero_bits << 16);
  if (lane < rq / 4) reinterpret_cast<uint32_t*>(rec_out)[lane] = mine;
}

// Compress one fp16 token vector (raw = this lane's 4 channels, already loaded) into record
// `rec` (a3): bitmaps, packed values + zero padding (or the 4-bit record when vbits == 4),
// tile offsets.
// kw: this unit's float32 channel weights for output-aware K pruning, or null (magnitude).
__device__ __forceinline__ void compress_raw_warp(uint2 raw, int k, int kpad, uint32_t rec,
                                                  uint64_t* __restrict__ bm_out, uint16_t* __restrict__ val_out,
                                                  uint32_t* __restrict__ off_out, int lane,
                                                  const float* __restrict__ kw = nullptr, int vbits = 16,
                                                  int rq = 0) {
  const uint32_t nib = kw ? select_keep_nibble_scored(raw.x, raw.y, reinterpret_cast<const float4*>(kw)[lane], (uint32_t)k)
                          : select_keep_nibble(raw.x, raw.y, (uint32_t)k, lane);
  // 128-bit keep mask: word i = channels 32i..32i+31 = lanes 8i..8i+7
  const int wi = lane >> 3, sh = 4 * (lane & 7);
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) w[i] = warp_or(wi == i ? (nib << sh) : 0u);
  const uint32_t wsel = wi == 0 ? w[0] : wi == 1 ? w[1] : wi == 2 ? w[2] : w[3];
  uint32_t pos = __popc(wsel & ((1u << sh) - 1u));
#pragma unroll
  for (int i = 0; i < 3; ++i) pos += (i < wi) ? __popc(w[i]) : 0u;
  const uint32_t h[4] = {raw.x & 0xFFFFu, raw.x >> 16, raw.y & 0xFFFFu, raw.y >> 16};
  if (vbits == 4) {
    quantize_token_warp(h, nib, pos, k, rq, reinterpret_cast<uint8_t*>(val_out), lane);
  } else {
    uint32_t p = pos;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (nib & (1u << j)) val_out[p++] = (uint16_t)h[j];
    }
    if (lane < kpad - k) val_out[k + lane] = 0;  // zero padding
  }
  if (lane == 0) {
    *reinterpret_cast<uint4*>(bm_out) = make_uint4(w[0], w[1], w[2], w[3]);  // tile0 = w0 | w1 << 32
    const uint32_t base = rec * (uint32_t)kpad;
    *reinterpret_cast<uint2*>(off_out) = make_uint2(base, base + __popc(w[0]) + __popc(w[1]));
  }
}

// Compress one fp16 token vector `src` (device, 8B-aligned, kD halves) into record `rec`.
__device__ __forceinline__ void compress_token_warp(const uint16_t* __restrict__ src, int k, int kpad,
                                                    uint32_t rec, uint64_t* __restrict__ bm_out,
                                                    uint16_t* __restrict__ val_out,
                                                    uint32_t* __restrict__ off_out, int lane,
                                                    const float* __restrict__ kw = nullptr, int vbits = 16,
                                                    int rq = 0) {
  const uint2 raw = *reinterpret_cast<const uint2*>(src + 4 * lane);
  compress_raw_warp(raw, k, kpad, rec, bm_out, val_out, off_out, lane, kw, vbits, rq);
}

__device__ __forceinline__ void copy_token_warp(const uint16_t* __restrict__ src, uint16_t* __restrict__ dst,
                                                int lane) {
  reinterpret_cast<uint2*>(dst)[lane] = reinterpret_cast<const uint2*>(src)[lane];
}

struct Sel {
  uint64_t* bm; uint16_t* val; uint32_t* off; uint16_t* win; int keep, kpad, rq;
  // value record of record index rec (fp16 values or the 4-bit record)
  __device__ __forceinline__ uint16_t* rec_val(size_t rec) const {
    return reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(val) + rec * (size_t)rq);
  }
};
__device__ __forceinline__ Sel sel_tensor(const CacheView& c, int x) {
  Sel r;
  r.bm = x ? c.bm[1] : c.bm[0];
  r.val = x ? c.val[1] : c.val[0];
  r.off = x ? c.off[1] : c.off[0];
  r.win = x ? c.win[1] : c.win[0];
  r.keep = x ? c.keep[1] : c.keep[0];
  r.kpad = x ? c.kpad[1] : c.kpad[0];
  r.rq = x ? c.rq[1] : c.rq[0];
  return r;
}

// a4 for one tensor (x = 0: K, 1: V) of unit u, one warp: with a full window the
// oldest window token is compressed into record nc and the new token takes its ring slot;
// otherwise the new token is appended to the ring (W == 0: compressed directly). nc, nw are
// the unit's counters before the append; the caller updates them.
__device__ __forceinline__ void append_unit_warp(const CacheView& c, int x, int u, const uint16_t* __restrict__ src,
                                                 int nc, int nw, int lane) {
  const size_t rec = (size_t)u * c.cap + nc;
  const Sel z = sel_tensor(c, x);
  const float* kw = (x == 0 && c.kw) ? c.kw + (size_t)u * kD : nullptr;
  const uint2 tok = reinterpret_cast<const uint2*>(src)[lane];  // the new token (load issued first)
  if (c.W == 0) {
    compress_raw_warp(tok, z.keep, z.kpad, (uint32_t)nc, z.bm + rec * kTiles, z.rec_val(rec),
                      z.off + rec * kTiles, lane, kw, c.vbits, z.rq);
  } else if (nw == c.W) {
    uint2* slot = reinterpret_cast<uint2*>(z.win + ((size_t)u * c.W + (nc % c.W)) * kD);
    const uint2 old = slot[lane];  // the evicted (oldest) window token
    compress_raw_warp(old, z.keep, z.kpad, (uint32_t)nc, z.bm + rec * kTiles, z.rec_val(rec),
                      z.off + rec * kTiles, lane, kw, c.vbits, z.rq);
    __syncwarp();
    slot[lane] = tok;
  } else {
    reinterpret_cast<uint2*>(z.win + ((size_t)u * c.W + ((nc + nw) % c.W)) * kD)[lane] = tok;
  }
}

}  // namespace mstf
