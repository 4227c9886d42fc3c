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
#include "compress_dev.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace mstf {

__global__ void set_counters_uniform(int32_t* n_comp, int32_t* n_win, int U, int nc, int nw) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < U) {
    n_comp[u] = nc;
    n_win[u] = nw;
  }
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
  append_unit_warp(c, x, u, (x ? v_new : k_new) + (size_t)u * kD, nc, nw, lane);
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
