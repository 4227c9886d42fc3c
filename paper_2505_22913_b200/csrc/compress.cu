// compress.cu -- K1: runtime per-token magnitude pruning + bitmap compression.
//
// One warp per token vector (d = 128, lane l owns channels 4l..4l+3, one 8-byte load).
//   a1  magnitude key  mag_c = bits_c & 0x7FFF (R3: fp16 magnitude as an unsigned integer)
//   a2  top-k select   tau = the k-th largest magnitude, found by a 15-step bisection on the
//                      magnitude bits with one redux.sync per step; channels with
//                      mag > tau are kept, and among mag == tau the (k - #{mag > tau})
//                      HIGHEST channel indices (ties prune the lower index first, R2)
//   a3  bitmap + pack  4 redux.or build the 128-bit keep mask (bit c <-> channel c, R6),
//                      popcount prefix sums give each kept value its packed slot, padding
//                      slots [k, kpad) are 0x0000 (R7), tile offsets p*kpad + popc(tiles<j) (R8)
// P:62 / P:173 (per-token magnitude pruning of K and V), P:218 (bitmap format)
// (prefill-then-compress, evict-on-exit), P:441 (multiples-of-8 padding).
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

__global__ void set_counters_uniform(int32_t* n_comp, int32_t* n_win, int U, int nc, int nw) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < U) {
    n_comp[u] = nc;
    n_win[u] = nw;
  }
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

// Bulk (prefill) mode: warp job j -> (tensor, unit, token). Counters were set beforehand.
__global__ void __launch_bounds__(256) prefill_kernel(CacheView c, const uint16_t* __restrict__ k,
                                                      const uint16_t* __restrict__ v, int T) {
  const int lane = threadIdx.x & 31;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long per_tensor = (long long)c.U * T;
  for (long long job = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); job < 2 * per_tensor;
       job += nwarps) {
    const int x = job >= per_tensor;  // 0 = K, 1 = V
    const long long r = job - x * per_tensor;
    const int u = (int)(r / T), t = (int)(r % T);
    const int nc = c.n_comp[u], nw = c.n_win[u];
    if (t >= nc + nw) continue;
    const uint16_t* src = (x ? v : k) + ((long long)u * T + t) * kD;
    const Sel z = sel_tensor(c, x);
    if (t < nc) {
      const size_t rec = (size_t)u * c.cap + t;
      compress_token_warp(src, z.keep, z.kpad, (uint32_t)t, z.bm + rec * kTiles, z.val + rec * z.kpad,
                          z.off + rec * kTiles, lane);
    } else {
      copy_token_warp(src, z.win + ((size_t)u * c.W + (t % c.W)) * kD, lane);
    }
  }
}

// Append (decode) mode: block = 2 warps (K, V) per unit.
__global__ void __launch_bounds__(64) append_kernel(CacheView c, const uint16_t* __restrict__ k_new,
                                                    const uint16_t* __restrict__ v_new) {
  const int u = blockIdx.x, x = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_launch_dependents();
  pdl_wait();  // the token and the counters may come from the previous kernel in the stream
  const int nc = c.n_comp[u], nw = c.n_win[u];
  const uint16_t* src = (x ? v_new : k_new) + (size_t)u * kD;
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
  __syncthreads();
  if (threadIdx.x == 0) {
    if (c.W == 0 || nw == c.W)
      c.n_comp[u] = nc + 1;
    else
      c.n_win[u] = nw + 1;
  }
}

cudaError_t launch_set_counters(const CacheView& c, const int32_t* nc_host, const int32_t* nw_host,
                                int32_t uniform_T, cudaStream_t s) {
  if (nc_host == nullptr) {
    const int nw = uniform_T < c.W ? uniform_T : c.W;
    set_counters_uniform<<<(c.U + 255) / 256, 256, 0, s>>>(c.n_comp, c.n_win, c.U, uniform_T - nw, nw);
    return cudaGetLastError();
  }
  cudaError_t e = cudaMemcpyAsync(c.n_comp, nc_host, sizeof(int32_t) * c.U, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  return cudaMemcpyAsync(c.n_win, nw_host, sizeof(int32_t) * c.U, cudaMemcpyHostToDevice, s);
}

cudaError_t launch_prefill(const CacheView& c, const uint16_t* k, const uint16_t* v, int32_t T,
                           cudaStream_t s) {
  if (T == 0 || c.U == 0) return cudaSuccess;
  const long long jobs = 2LL * c.U * T;
  long long blocks = (jobs + 7) / 8;
  if (blocks > 148LL * 64) blocks = 148LL * 64;
  prefill_kernel<<<(int)blocks, 256, 0, s>>>(c, k, v, T);
  return cudaGetLastError();
}

cudaError_t launch_append(const CacheView& c, const uint16_t* k_new, const uint16_t* v_new, cudaStream_t s) {
  return launch_pdl(append_kernel, dim3(c.U), dim3(64), 0, s, c, k_new, v_new);
}

}  // namespace mstf
