// compress_dev.cuh -- device code of K1 (per-token magnitude pruning + bitmap compression)
// shared by compress.cu (prefill / append kernels) and attention.cu (fused decode step).
// See compress.cu for the method and its citations.
#pragma once
#include <cstdint>

#include "kernels.cuh"
#include "ptx.cuh"

namespace mstf {

// Compress one fp16 token vector `src` (device, 8B-aligned, kD halves) into record `rec`.
__device__ __forceinline__ void compress_token_warp(const uint16_t* __restrict__ src, int k, int kpad,
                                                    uint32_t rec, uint64_t* __restrict__ bm_out,
                                                    uint16_t* __restrict__ val_out,
                                                    uint32_t* __restrict__ off_out, int lane) {
  const uint2 raw = *reinterpret_cast<const uint2*>(src + 4 * lane);
  uint32_t h[4] = {raw.x & 0xFFFFu, raw.x >> 16, raw.y & 0xFFFFu, raw.y >> 16};
  uint32_t m[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) m[j] = h[j] & 0x7FFFu;

  // tau = max t such that #{c : mag_c >= t} >= k   (count is non-increasing in t)
  uint32_t tau = 0;
#pragma unroll
  for (int b = 14; b >= 0; --b) {
    const uint32_t cand = tau | (1u << b);
    uint32_t c = (m[0] >= cand) + (m[1] >= cand) + (m[2] >= cand) + (m[3] >= cand);
    c = __reduce_add_sync(0xffffffffu, c);
    if (c >= (uint32_t)k) tau = cand;
  }
  uint32_t gt = (m[0] > tau) + (m[1] > tau) + (m[2] > tau) + (m[3] > tau);
  gt = __reduce_add_sync(0xffffffffu, gt);
  const uint32_t need = (uint32_t)k - gt;  // >= 1 slots for channels with mag == tau

  // ties: keep the `need` highest channel indices among mag == tau
  const uint32_t gtm = lanemask_gt();
  uint32_t above = 0;
  bool eq[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    eq[j] = (m[j] == tau);
    above += __popc(__ballot_sync(0xffffffffu, eq[j]) & gtm);
  }
  uint32_t nib = 0;
#pragma unroll
  for (int j = 3; j >= 0; --j) {
    const bool keep = (m[j] > tau) || (eq[j] && above < need);
    if (eq[j]) ++above;
    nib |= (uint32_t)keep << j;
  }

  // 128-bit keep mask: word i = channels 32i..32i+31 = lanes 8i..8i+7
  const int wi = lane >> 3, sh = 4 * (lane & 7);
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) w[i] = __reduce_or_sync(0xffffffffu, wi == i ? (nib << sh) : 0u);

  const uint32_t wsel = wi == 0 ? w[0] : wi == 1 ? w[1] : wi == 2 ? w[2] : w[3];
  uint32_t pos = __popc(wsel & ((1u << sh) - 1u));
#pragma unroll
  for (int i = 0; i < 3; ++i) pos += (i < wi) ? __popc(w[i]) : 0u;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (nib & (1u << j)) val_out[pos++] = (uint16_t)h[j];
  }
  if (lane < kpad - k) val_out[k + lane] = 0;  // zero padding
  if (lane == 0) {
    const uint4 bmw = make_uint4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<uint4*>(bm_out) = bmw;  // little endian: tile0 = w0 | w1 << 32
    const uint32_t base = rec * (uint32_t)kpad;
    *reinterpret_cast<uint2*>(off_out) = make_uint2(base, base + __popc(w[0]) + __popc(w[1]));
  }
}

__device__ __forceinline__ void copy_token_warp(const uint16_t* __restrict__ src, uint16_t* __restrict__ dst,
                                                int lane) {
  reinterpret_cast<uint2*>(dst)[lane] = reinterpret_cast<const uint2*>(src)[lane];
}

struct Sel {
  uint64_t* bm; uint16_t* val; uint32_t* off; uint16_t* win; int keep, kpad;
};
__device__ __forceinline__ Sel sel_tensor(const CacheView& c, int x) {
  Sel r;
  r.bm = x ? c.bm[1] : c.bm[0];
  r.val = x ? c.val[1] : c.val[0];
  r.off = x ? c.off[1] : c.off[0];
  r.win = x ? c.win[1] : c.win[0];
  r.keep = x ? c.keep[1] : c.keep[0];
  r.kpad = x ? c.kpad[1] : c.kpad[0];
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
  if (c.W == 0) {
    compress_token_warp(src, z.keep, z.kpad, (uint32_t)nc, z.bm + rec * kTiles, z.val + rec * z.kpad,
                        z.off + rec * kTiles, lane);
  } else if (nw == c.W) {
    uint16_t* slot = z.win + ((size_t)u * c.W + (nc % c.W)) * kD;
    compress_token_warp(slot, z.keep, z.kpad, (uint32_t)nc, z.bm + rec * kTiles, z.val + rec * z.kpad,
                        z.off + rec * kTiles, lane);
    __syncwarp();
    copy_token_warp(src, slot, lane);
  } else {
    copy_token_warp(src, z.win + ((size_t)u * c.W + ((nc + nw) % c.W)) * kD, lane);
  }
}

}  // namespace mstf
