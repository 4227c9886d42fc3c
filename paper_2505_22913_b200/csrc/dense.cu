// dense.cu -- the dense-KV decode baseline (the comparison of P:439 / P:458, on the repo's own
// mma.sync skeleton), the cross-shard merge of the sequence split (NEXT-3), and the stream-K
// cost model shared by the host planner and attn_warp.cu.
//
// Dense kernel: grid (splits, U), 4 warps per CTA, each warp a strided set of 16-token blocks of
// one unit; fragments straight from 128-bit global loads (no expansion); scores S^T[16 tok x 8
// heads] = K_blk . q^T (a5/a6, mma.sync m16n8k16, fp32 accumulate), online softmax (a7, exp2),
// O^T[128 ch x 8 heads] += V_blk^T . P^T (a8) with the even / odd channels in two MMAs; one
// partial per warp, merged by mstf_combine_kernel (a9).
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "kernels.cuh"
#include "ptx.cuh"

namespace mstf {
// 2^x with the single MUFU.EX2 (ex2.approx.ftz): the arguments are s - max <= 0, results in
// (0, 1]; results below 2^-126 flush to 0 (weights that small do not change an fp32 sum of
// terms >= 1). exp2f adds a range check and two multiplies per call for subnormal results.
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---------------------------------------------------------------- smem helpers
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
// Per-block register operands, already expanded (zeros at pruned channels):
//   k[r][j] : token g (r=0) / g+8 (r=1), channels 32t+2j, 32t+2j+1   (K mma A operand)
//   v[x][j] : token {2t, 2t+1, 2t+8, 2t+9}[x], channels 16g+2j, 16g+2j+1 (V mma A operand)
struct BlockRegs {
  uint32_t k[2][16];
  uint32_t v[4][8];
};
// ---------------------------------------------------------------- dense source
// 16 dense token rows of fp16 [*, kD] in global memory (window ring / dense KV baseline).
struct DenseBlock {
  const uint16_t* k;
  const uint16_t* v;
  int row0, nvalid;
  bool ring;           // window ring: slots row0..row0+15 of a W-slot ring whose oldest
  int W, first, nwin;  // token sits in slot `first` and which holds `nwin` tokens
  __device__ __forceinline__ bool valid(int r) const {
    const int slot = row0 + r;
    if (!ring) return r < nvalid;
    int age = slot - first;  // ring position relative to the oldest token, in [0, W)
    if (age < 0) age += W;
    return slot < W && age < nwin;
  }
};

__device__ __forceinline__ void fill_dense(const DenseBlock& db, BlockRegs& r, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    const int tok = g + 8 * x;
    if (db.valid(tok)) {
      const uint4* p = reinterpret_cast<const uint4*>(db.k + (size_t)(db.row0 + tok) * kD + 32 * t);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 a = p[i];
        r.k[x][4 * i] = a.x; r.k[x][4 * i + 1] = a.y; r.k[x][4 * i + 2] = a.z; r.k[x][4 * i + 3] = a.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) r.k[x][i] = 0;
    }
  }
  const int tk[4] = {2 * t, 2 * t + 1, 2 * t + 8, 2 * t + 9};
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    if (db.valid(tk[x])) {
      const uint4* p = reinterpret_cast<const uint4*>(db.v + (size_t)(db.row0 + tk[x]) * kD + 16 * g);
      const uint4 a = p[0], b = p[1];
      r.v[x][0] = a.x; r.v[x][1] = a.y; r.v[x][2] = a.z; r.v[x][3] = a.w;
      r.v[x][4] = b.x; r.v[x][5] = b.y; r.v[x][6] = b.z; r.v[x][7] = b.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) r.v[x][i] = 0;
    }
  }
}

// Per-warp online-softmax attention state.
struct WarpState {
  float acc[2][4][4];  // [channel parity e][m-tile i]: rows ch 16g+2i+e | 16g+8+2i+e, cols heads 2t, 2t+1
  float m0, m1, l0, l1;
  uint32_t qf[16];     // q of head g, channels 32t..32t+31 (half2 pairs)
};

// a5 + a7 + a8 for one block of 16 tokens (first/last validity via `vg`, `vg8`).
__device__ __forceinline__ void process_block(const BlockRegs& r, bool vg, bool vg8, WarpState& st,
                                              float scale_log2) {
  // ---- a5: scores S^T[tok][head] (rows tokens g, g+8; cols heads 2t, 2t+1)
  float sc[4] = {0.f, 0.f, 0.f, 0.f}, sd[4] = {0.f, 0.f, 0.f, 0.f};  // two chains hide HMMA latency
#pragma unroll
  for (int s = 0; s < 8; s += 2) {
    mma16816(sc, r.k[0][2 * s], r.k[1][2 * s], r.k[0][2 * s + 1], r.k[1][2 * s + 1], st.qf[2 * s], st.qf[2 * s + 1]);
    mma16816(sd, r.k[0][2 * s + 2], r.k[1][2 * s + 2], r.k[0][2 * s + 3], r.k[1][2 * s + 3], st.qf[2 * s + 2],
             st.qf[2 * s + 3]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) sc[i] += sd[i];
  // ---- a7: online softmax (log2 domain)
  const float x0 = vg ? sc[0] * scale_log2 : -INFINITY;
  const float x1 = vg ? sc[1] * scale_log2 : -INFINITY;
  const float x2 = vg8 ? sc[2] * scale_log2 : -INFINITY;
  const float x3 = vg8 ? sc[3] * scale_log2 : -INFINITY;
  float bm0 = fmaxf(x0, x2), bm1 = fmaxf(x1, x3);
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, o));
    bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, o));
  }
  const float mn0 = fmaxf(st.m0, bm0), mn1 = fmaxf(st.m1, bm1);
  const float a0 = fast_exp2(st.m0 - mn0), a1 = fast_exp2(st.m1 - mn1);
  const float p0 = fast_exp2(x0 - mn0), p1 = fast_exp2(x1 - mn1), p2 = fast_exp2(x2 - mn0), p3 = fast_exp2(x3 - mn1);
  st.l0 = st.l0 * a0 + (p0 + p2);
  st.l1 = st.l1 * a1 + (p1 + p3);
  st.m0 = mn0;
  st.m1 = mn1;
  if (__any_sync(0xffffffffu, a0 != 1.f || a1 != 1.f)) {
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        st.acc[e][i][0] *= a0; st.acc[e][i][1] *= a1; st.acc[e][i][2] *= a0; st.acc[e][i][3] *= a1;
      }
  }
  // ---- P^T: lane (g,t) gets (p[2t][g], p[2t+1][g]) (kappa 0) and tokens 2t+8, 2t+9 (kappa 1)
  const uint32_t m[2] = {movmatrix_t(pack_half2(p0, p1)), movmatrix_t(pack_half2(p2, p3))};
  // ---- a8: O^T[ch pair rows][heads] += V-pairs . P, split into even / odd channels
#pragma unroll
  for (int kap = 0; kap < 2; ++kap) {
    const uint32_t be0 = m[kap] & 0xFFFFu, be1 = m[kap] >> 16, bo0 = m[kap] << 16, bo1 = m[kap] & 0xFFFF0000u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t a0r = r.v[2 * kap][i], a1r = r.v[2 * kap][4 + i];
      const uint32_t a2r = r.v[2 * kap + 1][i], a3r = r.v[2 * kap + 1][4 + i];
      mma16816(st.acc[0][i], a0r, a1r, a2r, a3r, be0, be1);
      mma16816(st.acc[1][i], a0r, a1r, a2r, a3r, bo0, bo1);
    }
  }
}

// K-warp state and block step: scores + online softmax; returns the V-warp handoff
__device__ __forceinline__ void init_state(WarpState& st, const uint16_t* q_unit, int G, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int e = 0; e < 2; ++e)
#pragma unroll
    for (int i = 0; i < 4; ++i) st.acc[e][i][0] = st.acc[e][i][1] = st.acc[e][i][2] = st.acc[e][i][3] = 0.f;
  st.m0 = st.m1 = -INFINITY;
  st.l0 = st.l1 = 0.f;
  if (g < G) {
    const uint4* p = reinterpret_cast<const uint4*>(q_unit + g * kD + 32 * t);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 x = p[i];
      st.qf[4 * i] = x.x; st.qf[4 * i + 1] = x.y; st.qf[4 * i + 2] = x.z; st.qf[4 * i + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) st.qf[i] = 0;
  }
}

// Write this warp's partial (m, l in log2 domain; o unnormalised).
__device__ __forceinline__ void store_partial(WarpState& st, float* ws_o, float* ws_ml, size_t pidx, int G,
                                              int lane) {
  const int g = lane >> 2, t = lane & 3;
  float l0 = st.l0, l1 = st.l1;
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, o);
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  }
  float* o = ws_o + pidx * G * kD;
  float* ml = ws_ml + pidx * G * 2;
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const int h = 2 * t + hh;
    if (h < G) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        *reinterpret_cast<float2*>(o + h * kD + 16 * g + 2 * i) = make_float2(st.acc[0][i][hh], st.acc[1][i][hh]);
        *reinterpret_cast<float2*>(o + h * kD + 16 * g + 8 + 2 * i) =
            make_float2(st.acc[0][i][2 + hh], st.acc[1][i][2 + hh]);
      }
      if (g == 0) {
        ml[2 * h] = hh ? st.m1 : st.m0;
        ml[2 * h + 1] = hh ? l1 : l0;
      }
    }
  }
}

// ---------------------------------------------------------------- K2 (K/V warp-specialised)
// 4 K-warps (0..3) + 4 V-warps (4..7) + 1 producer warp (8). K-warp w and V-warp w+4 share the
// tokens [16w, 16w+16) of every stage: the K-warp gathers K, computes scores and the online
// softmax and hands {P^T fragments, rescale factors} to its V-warp through a 2-slot shared
// ---------------------------------------------------------------- K3: combine partials
__global__ void mstf_combine_kernel(const float* __restrict__ ws_o, const float* __restrict__ ws_ml, int nparts,
                                    int G, void* out, int out_f16, float* part_ml, float* part_o) {
  pdl_launch_dependents();
  pdl_wait();  // partials come from the attention kernel just before
  // one warp per (unit, head); lane owns channels 4*lane .. 4*lane+3
  const int u = blockIdx.x, h = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (h >= G) return;
  float M = -INFINITY;
  for (int i = lane; i < nparts; i += 32) M = fmaxf(M, ws_ml[(((size_t)u * nparts + i) * G + h) * 2]);
#pragma unroll
  for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  float L = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
  for (int i = 0; i < nparts; ++i) {
    const size_t pi = (size_t)u * nparts + i;
    const float2 ml = *reinterpret_cast<const float2*>(ws_ml + (pi * G + h) * 2);
    const float4 o = *reinterpret_cast<const float4*>(ws_o + (pi * G + h) * kD + 4 * lane);
    const float w = ml.x == -INFINITY ? 0.f : exp2f(ml.x - M);
    L += w * ml.y;
    acc.x += w * o.x; acc.y += w * o.y; acc.z += w * o.z; acc.w += w * o.w;
  }
  const size_t oi = ((size_t)u * G + h) * kD + 4 * lane;
  if (part_ml) {  // sequence-split shard: unnormalised partials (log2 domain)
    *reinterpret_cast<float4*>(part_o + oi) = acc;
    if (lane == 0) *reinterpret_cast<float2*>(part_ml + ((size_t)u * G + h) * 2) = make_float2(M, L);
    return;
  }
  const float inv = 1.f / L;
  if (out_f16) {
    __half2* po = reinterpret_cast<__half2*>(reinterpret_cast<__half*>(out) + oi);
    po[0] = __floats2half2_rn(acc.x * inv, acc.y * inv);
    po[1] = __floats2half2_rn(acc.z * inv, acc.w * inv);
  } else {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + oi) =
        make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  }
}

// Sequence-split merge (NEXT-3): n shards' partials [n][U][G] (m in log2 units, l, o unnormalised)
// -> O = sum_i 2^(m_i - M) o_i / sum_i 2^(m_i - M) l_i, the a9 combine across shards. One warp per
// (unit, head); an all-empty (unit, head) (L = 0) gives 0.
__global__ void mstf_merge_kernel(int n, int U, int G, const float* __restrict__ ml, const float* __restrict__ o,
                                  void* out, int out_f16) {
  const int u = blockIdx.x, h = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (h >= G) return;
  float M = -INFINITY;
  for (int i = lane; i < n; i += 32) M = fmaxf(M, ml[(((size_t)i * U + u) * G + h) * 2]);
#pragma unroll
  for (int s = 16; s; s >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, s));
  float L = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = 0; i < n; ++i) {
    const size_t pi = ((size_t)i * U + u) * G + h;
    const float2 m = *reinterpret_cast<const float2*>(ml + pi * 2);
    const float4 v = *(reinterpret_cast<const float4*>(o + pi * kD) + lane);
    const float w = m.x == -INFINITY ? 0.f : exp2f(m.x - M);
    L += w * m.y;
    acc.x += w * v.x; acc.y += w * v.y; acc.z += w * v.z; acc.w += w * v.w;
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  const size_t oi = ((size_t)u * G + h) * kD + 4 * lane;
  if (out_f16) {
    __half2* po = reinterpret_cast<__half2*>(reinterpret_cast<__half*>(out) + oi);
    po[0] = __floats2half2_rn(acc.x * inv, acc.y * inv);
    po[1] = __floats2half2_rn(acc.z * inv, acc.w * inv);
  } else {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + oi) =
        make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  }
}

// The partials of a shard without tokens: m = -inf, l = 0, o = 0 (the merge's identity).
__global__ void mstf_empty_partial_kernel(float* __restrict__ ml, float* __restrict__ o, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    reinterpret_cast<float2*>(ml)[i] = make_float2(-INFINITY, 0.f);
    float4* po = reinterpret_cast<float4*>(o + (size_t)i * kD);
#pragma unroll
    for (int j = 0; j < kD / 4; ++j) po[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

cudaError_t launch_empty_partials(float* ml, float* o, int32_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  mstf_empty_partial_kernel<<<(n + 127) / 128, 128, 0, s>>>(ml, o, n);
  return cudaGetLastError();
}

cudaError_t launch_merge_partials(int32_t n, int32_t U, int32_t G, const float* ml, const float* o, void* out,
                                  int32_t out_f16, cudaStream_t s) {
  if (U == 0) return cudaSuccess;
  mstf_merge_kernel<<<U, G * 32, 0, s>>>(n, U, G, ml, o, out, out_f16);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- dense baseline
__global__ void __launch_bounds__(kConsumerWarps * 32) mstf_dense_attn_kernel(
    const uint16_t* __restrict__ k, const uint16_t* __restrict__ v, const int32_t* __restrict__ lengths,
    int t_max, const uint16_t* __restrict__ q, int G, float scale_log2, float* ws_o, float* ws_ml) {
  const int u = blockIdx.y, split = blockIdx.x, S = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = lengths[u];
  const int blocks_total = (n + 15) / 16;
  const int per = (blocks_total + S - 1) / S;
  const int b0 = min(split * per, blocks_total), b1 = min(b0 + per, blocks_total);
  WarpState st;
  init_state(st, q + (size_t)u * G * kD, G, lane);
  for (int b = b0 + warp; b < b1; b += kConsumerWarps) {
    DenseBlock db;
    db.k = k + (size_t)u * t_max * kD;
    db.v = v + (size_t)u * t_max * kD;
    db.ring = false;
    db.W = db.first = db.nwin = 0;
    db.row0 = b * 16;
    db.nvalid = min(16, n - b * 16);
    BlockRegs r;
    fill_dense(db, r, lane);
    process_block(r, db.valid(lane >> 2), db.valid((lane >> 2) + 8), st, scale_log2);
  }
  store_partial(st, ws_o, ws_ml, ((size_t)u * S + split) * kConsumerWarps + warp, G, lane);
}


// ---------------------------------------------------------------- host side
void sk_cost_params(int32_t* cs, int32_t* cw) {
  static const int32_t s_cs = std::getenv("MSTF_SKCS") ? std::atoi(std::getenv("MSTF_SKCS")) : 2;
  static const int32_t s_cw = std::getenv("MSTF_SKCW") ? std::max(1, std::atoi(std::getenv("MSTF_SKCW"))) : 2;
  *cs = s_cs;
  *cw = s_cw;
}

int32_t sk_unit_cost(int32_t n_comp, int32_t W) {
  int32_t cs, cw;
  sk_cost_params(&cs, &cw);
  return cs + (n_comp + 15) / 16 + (W > 0 ? (W + 15) / 16 : 0) * cw;
}

size_t dense_ws_bytes(int32_t U, int32_t G, int32_t splits) {
  const size_t parts = (size_t)U * splits * kConsumerWarps;
  return parts * G * (kD + 2) * sizeof(float) + 256;
}

cudaError_t launch_dense_attention(const uint16_t* k, const uint16_t* v, const int32_t* lengths, int32_t U,
                                   int32_t G, int32_t t_max, int32_t splits, const uint16_t* q, float scale,
                                   void* out, int32_t out_f16, void* ws, cudaStream_t s) {
  const size_t parts = (size_t)U * splits * kConsumerWarps;
  float* ws_o = reinterpret_cast<float*>(ws);
  float* ws_ml = ws_o + parts * G * kD;
  mstf_dense_attn_kernel<<<dim3(splits, U), kConsumerWarps * 32, 0, s>>>(k, v, lengths, t_max, q, G,
                                                                        scale * 1.4426950408889634f, ws_o, ws_ml);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  mstf_combine_kernel<<<U, G * 32, 0, s>>>(ws_o, ws_ml, splits * kConsumerWarps, G, out, out_f16, nullptr, nullptr);
  return cudaGetLastError();
}

}  // namespace mstf
