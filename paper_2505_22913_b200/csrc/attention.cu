// attention.cu -- K2/K3: split-sequence decode attention directly over the compressed
// cache (Algorithm 1), and the dense-KV baseline on the same skeleton.
//
// K2 (mstf_attn_kernel), grid = (splits, U), block = 4 consumer warps + 1 producer warp.
//   * producer (one lane): streams the split's compressed records chunk by chunk
//     (kChunk tokens: K bitmaps, K values, V bitmaps, V values -- four contiguous
//     cp.async.bulk copies) into an nstage-deep shared-memory ring guarded by mbarriers
//     (full: tx-count, empty: one arrive per consumer warp).
//   * consumer warp w takes tokens [16w, 16w+16) of every chunk:
//       a5  S^T[16 tok x 8 heads] = K_blk[16 x 128] . q^T   -- 8 x mma.m16n8k16; the A
//           operand is the K block expanded from (bitmap, packed values) in registers
//           ("load-as-compressed, compute-as-dense"), zeros at pruned channels
//       a7  online softmax (running max m, sum l per head, exp2 with log2e folded in)
//       a8  O^T[128 ch x 8 heads] += V_blk^T[128 x 16] . P^T[16 x 8]  -- 8 x mma; P^T is
//           the score accumulator converted to fp16 and transposed with movmatrix
//     the last split also covers the dense local window (a6, Alg. 1 lines 1 and 5).
//   * each warp writes its (m, l, o) partial to the workspace.
// K3 (mstf_combine_kernel): per (unit, head, channel), merges the partials (a9).
//
// Fragment <-> channel mapping (free permutations of the contraction / output index):
//   K mma, lane (g = lane/4, t = lane%4): tokens g and g+8, channels 32t..32t+31
//     (= bitmap word t of the token); k-step s uses channels 32t+4s+{0,1} (a0/a1, b0)
//     and 32t+4s+{2,3} (a2/a3, b1).
//   V mma, m-tile i: row r <-> channel 8r+i, i.e. lane (g,t) expands bitmap bytes g and
//     g+8 of tokens 2t, 2t+1, 2t+8, 2t+9.
#include <cfloat>
#include <cmath>

#include "kernels.cuh"
#include "ptx.cuh"

namespace mstf {

constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kBarBytes = 128;  // 8 stages x {full, empty} x 8 B

struct AttnParams {
  CacheView c;
  const uint16_t* q;  // [U][G][kD]
  float* ws_o;        // [U][S][NW][G][kD]
  float* ws_ml;       // [U][S][NW][G][2]
  int G;
  float scale_log2;
  int nstage, stage_bytes;
  int off_kval, off_vbm, off_vval;  // byte offsets inside a stage (kbm at 0)
};

// ---------------------------------------------------------------- expansion helpers
// 32 channels of one token (bitmap word `w`, `pre` kept channels before it) from the packed
// values `vals` (shared or global) -> 16 half2 registers, zero at pruned channels.
__device__ __forceinline__ void expand_word(const uint16_t* __restrict__ vals, uint32_t w, uint32_t pre,
                                            uint32_t (&e)[16]) {
  const uint16_t* p = vals + pre;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t b0 = (w >> (2 * i)) & 1u, b1 = (w >> (2 * i + 1)) & 1u;
    const uint32_t lo = b0 ? (uint32_t)p[0] : 0u;
    p += b0;
    const uint32_t hi = b1 ? (uint32_t)p[0] : 0u;
    p += b1;
    e[i] = lo | (hi << 16);
  }
}

// 8 channels (bitmap byte `byte`, `pre` kept channels before it) -> 8 halves in out[0..7].
__device__ __forceinline__ void expand_byte(const uint16_t* __restrict__ vals, uint32_t byte, uint32_t pre,
                                            uint32_t (&out)[8]) {
  const uint16_t* p = vals + pre;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t b = (byte >> i) & 1u;
    out[i] = b ? (uint32_t)p[0] : 0u;
    p += b;
  }
}

__device__ __forceinline__ uint32_t popc_before_word(const uint4& bw, int t) {
  return (t > 0 ? __popc(bw.x) : 0) + (t > 1 ? __popc(bw.y) : 0) + (t > 2 ? __popc(bw.z) : 0);
}
__device__ __forceinline__ uint32_t word_of(const uint4& bw, int t) {
  return t == 0 ? bw.x : t == 1 ? bw.y : t == 2 ? bw.z : bw.w;
}

// Compressed block source: 16 tokens of a stage in shared memory.
struct CompSrc {
  const uint4* kbm;      // [kChunk] 16-byte bitmap records
  const uint16_t* kval;  // [kChunk][kpk]
  const uint4* vbm;
  const uint16_t* vval;
  int kpk, kpv, tok0, nvalid;  // tokens tok0..tok0+15 of the stage, first nvalid valid

  __device__ __forceinline__ bool valid(int r) const { return r < nvalid; }
  __device__ __forceinline__ void load_k(int r, int t, uint32_t (&e)[16]) const {
    uint4 bw = kbm[tok0 + r];
    if (!valid(r)) bw = make_uint4(0, 0, 0, 0);
    expand_word(kval + (tok0 + r) * kpk, word_of(bw, t), popc_before_word(bw, t), e);
  }
  // bytes g and g+8 of token r -> lo[8], hi[8]
  __device__ __forceinline__ void load_v(int r, int g, uint32_t (&lo)[8], uint32_t (&hi)[8]) const {
    uint4 bw = vbm[tok0 + r];
    if (!valid(r)) bw = make_uint4(0, 0, 0, 0);
    const uint16_t* vals = vval + (tok0 + r) * kpv;
    const int wl = g >> 2, sh = 8 * (g & 3);
    const uint32_t wlo = wl ? bw.y : bw.x, whi = wl ? bw.w : bw.z;
    const uint32_t below = (1u << sh) - 1u;
    const uint32_t pre_lo = (wl ? __popc(bw.x) : 0) + __popc(wlo & below);
    const uint32_t pre_hi = __popc(bw.x) + __popc(bw.y) + (wl ? __popc(bw.z) : 0) + __popc(whi & below);
    expand_byte(vals, (wlo >> sh) & 0xFFu, pre_lo, lo);
    expand_byte(vals, (whi >> sh) & 0xFFu, pre_hi, hi);
  }
};

// Dense block source: 16 token rows of fp16 [*, kD] in global memory (window / dense KV).
struct DenseSrc {
  const uint16_t* k;   // row pointer base; token r at k + row(r) * kD
  const uint16_t* v;
  int row0, nvalid;
  bool ring;           // window ring: slots row0..row0+15 of a W-slot ring whose oldest
  int W, first, nwin;  // token sits in slot `first` and which holds `nwin` tokens

  __device__ __forceinline__ int row(int r) const { return row0 + r; }
  __device__ __forceinline__ bool valid(int r) const {
    const int slot = row0 + r;
    return ring ? (slot < W && ((slot - first + W) % W) < nwin) : r < nvalid;
  }
  __device__ __forceinline__ void load_k(int r, int t, uint32_t (&e)[16]) const {
    if (!valid(r)) {
#pragma unroll
      for (int i = 0; i < 16; ++i) e[i] = 0;
      return;
    }
    const uint4* p = reinterpret_cast<const uint4*>(k + (size_t)row(r) * kD + 32 * t);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 x = p[i];
      e[4 * i] = x.x; e[4 * i + 1] = x.y; e[4 * i + 2] = x.z; e[4 * i + 3] = x.w;
    }
  }
  __device__ __forceinline__ void load_v(int r, int g, uint32_t (&lo)[8], uint32_t (&hi)[8]) const {
    if (!valid(r)) {
#pragma unroll
      for (int i = 0; i < 8; ++i) lo[i] = hi[i] = 0;
      return;
    }
    const uint16_t* base = v + (size_t)row(r) * kD;
    const uint4 a = *reinterpret_cast<const uint4*>(base + 8 * g);
    const uint4 b = *reinterpret_cast<const uint4*>(base + 64 + 8 * g);
    const uint32_t aa[4] = {a.x, a.y, a.z, a.w}, bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      lo[2 * i] = aa[i] & 0xFFFFu; lo[2 * i + 1] = aa[i] >> 16;
      hi[2 * i] = bb[i] & 0xFFFFu; hi[2 * i + 1] = bb[i] >> 16;
    }
  }
};

// Per-warp online-softmax attention state.
struct WarpState {
  float acc[8][4];  // O^T m-tile i: (ch 8g+i | 64+8g+i) x (heads 2t, 2t+1)
  float m0, m1, l0, l1;
  uint32_t qf[16];  // q of head g, channels 32t..32t+31 (half2 pairs)
};

// Process one block of 16 tokens from `src`.
template <class Src>
__device__ __forceinline__ void process_block(const Src& src, WarpState& st, float scale_log2, int lane) {
  const int g = lane >> 2, t = lane & 3;
  // ---- a5: scores S^T[tok][head]
  float sc[4] = {0.f, 0.f, 0.f, 0.f};
  {
    uint32_t eg[16], eg8[16];
    src.load_k(g, t, eg);
    src.load_k(g + 8, t, eg8);
#pragma unroll
    for (int s = 0; s < 8; ++s)
      mma16816(sc, eg[2 * s], eg8[2 * s], eg[2 * s + 1], eg8[2 * s + 1], st.qf[2 * s], st.qf[2 * s + 1]);
  }
  // ---- a7: online softmax (log2 domain)
  const bool vg = src.valid(g), vg8 = src.valid(g + 8);
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
  const float a0 = exp2f(st.m0 - mn0), a1 = exp2f(st.m1 - mn1);
  const float p0 = exp2f(x0 - mn0), p1 = exp2f(x1 - mn1), p2 = exp2f(x2 - mn0), p3 = exp2f(x3 - mn1);
  st.l0 = st.l0 * a0 + (p0 + p2);
  st.l1 = st.l1 * a1 + (p1 + p3);
  st.m0 = mn0;
  st.m1 = mn1;
  if (__any_sync(0xffffffffu, a0 != 1.f || a1 != 1.f)) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      st.acc[i][0] *= a0; st.acc[i][1] *= a1; st.acc[i][2] *= a0; st.acc[i][3] *= a1;
    }
  }
  // ---- P^T fragment (B operand of the V mma): head g, tokens 2t,2t+1 / 2t+8,2t+9
  const uint32_t pb0 = movmatrix_t(pack_half2(p0, p1));
  const uint32_t pb1 = movmatrix_t(pack_half2(p2, p3));
  // ---- a8: O^T += V^T P^T
  uint32_t A[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) A[i][0] = A[i][1] = A[i][2] = A[i][3] = 0;
  const int toks[4] = {2 * t, 2 * t + 1, 2 * t + 8, 2 * t + 9};
#pragma unroll
  for (int tk = 0; tk < 4; ++tk) {
    uint32_t lo[8], hi[8];
    src.load_v(toks[tk], g, lo, hi);
    const int sh = 16 * (tk & 1), base = (tk >> 1) * 2;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      A[i][base] |= lo[i] << sh;
      A[i][base + 1] |= hi[i] << sh;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) mma16816(st.acc[i], A[i][0], A[i][1], A[i][2], A[i][3], pb0, pb1);
}

__device__ __forceinline__ void init_state(WarpState& st, const uint16_t* q_unit, int G, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int i = 0; i < 8; ++i) st.acc[i][0] = st.acc[i][1] = st.acc[i][2] = st.acc[i][3] = 0.f;
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
  const int h0 = 2 * t, h1 = 2 * t + 1;
  float* o = ws_o + pidx * G * kD;
  float* ml = ws_ml + pidx * G * 2;
  if (h0 < G) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      o[h0 * kD + 8 * g + i] = st.acc[i][0];
      o[h0 * kD + 64 + 8 * g + i] = st.acc[i][2];
    }
    if (g == 0) { ml[2 * h0] = st.m0; ml[2 * h0 + 1] = l0; }
  }
  if (h1 < G) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      o[h1 * kD + 8 * g + i] = st.acc[i][1];
      o[h1 * kD + 64 + 8 * g + i] = st.acc[i][3];
    }
    if (g == 0) { ml[2 * h1] = st.m1; ml[2 * h1 + 1] = l1; }
  }
}

// ---------------------------------------------------------------- K2: sparse attention
__global__ void __launch_bounds__(kThreads) mstf_attn_kernel(const AttnParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 8;
  uint8_t* stages = smem + kBarBytes;

  const int u = blockIdx.y, split = blockIdx.x, S = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const CacheView& c = p.c;
  const int n = c.n_comp[u];
  const int chunks_total = (n + kChunk - 1) / kChunk;
  const int cps = (chunks_total + S - 1) / S;
  const int cbeg = min(split * cps, chunks_total), cend = min(cbeg + cps, chunks_total);
  const int nchunks = cend - cbeg;

  if (threadIdx.x == 0) {
    for (int i = 0; i < p.nstage; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ---------------- producer
    if (lane == 0) {
      const int kpk = c.kpad[0], kpv = c.kpad[1];
      const uint8_t* kbm = reinterpret_cast<const uint8_t*>(c.bm[0] + (size_t)u * c.cap * kTiles);
      const uint8_t* vbm = reinterpret_cast<const uint8_t*>(c.bm[1] + (size_t)u * c.cap * kTiles);
      const uint8_t* kval = reinterpret_cast<const uint8_t*>(c.val[0] + (size_t)u * c.cap * kpk);
      const uint8_t* vval = reinterpret_cast<const uint8_t*>(c.val[1] + (size_t)u * c.cap * kpv);
      for (int i = 0; i < nchunks; ++i) {
        const int st = i % p.nstage;
        if (i >= p.nstage) mbar_wait(&empty[st], ((i / p.nstage) - 1) & 1);
        const int tok0 = (cbeg + i) * kChunk;
        const int nt = min(kChunk, n - tok0);
        const uint32_t bbm = nt * 16, bk = nt * 2 * kpk, bv = nt * 2 * kpv;
        uint8_t* sb = stages + (size_t)st * p.stage_bytes;
        mbar_arrive_expect_tx(&full[st], 2 * bbm + bk + bv);
        bulk_g2s(sb, kbm + (size_t)tok0 * 16, bbm, &full[st]);
        bulk_g2s(sb + p.off_kval, kval + (size_t)tok0 * 2 * kpk, bk, &full[st]);
        bulk_g2s(sb + p.off_vbm, vbm + (size_t)tok0 * 16, bbm, &full[st]);
        bulk_g2s(sb + p.off_vval, vval + (size_t)tok0 * 2 * kpv, bv, &full[st]);
      }
    }
    return;
  }

  // ---------------- consumers
  WarpState st;
  init_state(st, p.q + (size_t)u * p.G * kD, p.G, lane);
  for (int i = 0; i < nchunks; ++i) {
    const int sidx = i % p.nstage;
    mbar_wait(&full[sidx], (i / p.nstage) & 1);
    const uint8_t* sb = stages + (size_t)sidx * p.stage_bytes;
    const int tok0 = (cbeg + i) * kChunk;
    const int nvalid = min(16, n - tok0 - 16 * warp);
    if (nvalid > 0) {
      CompSrc src;
      src.kbm = reinterpret_cast<const uint4*>(sb);
      src.kval = reinterpret_cast<const uint16_t*>(sb + p.off_kval);
      src.vbm = reinterpret_cast<const uint4*>(sb + p.off_vbm);
      src.vval = reinterpret_cast<const uint16_t*>(sb + p.off_vval);
      src.kpk = c.kpad[0];
      src.kpv = c.kpad[1];
      src.tok0 = 16 * warp;
      src.nvalid = nvalid;
      process_block(src, st, p.scale_log2, lane);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[sidx]);
  }
  // dense local window (Alg. 1 lines 1 and 5) on the last split
  if (split == S - 1 && c.W > 0) {
    const int nw = c.n_win[u];
    const int first = n % c.W;  // slot of the oldest window token (position n)
    for (int blk = warp; blk * 16 < c.W; blk += kConsumerWarps) {
      DenseSrc src;
      src.k = c.win[0] + (size_t)u * c.W * kD;
      src.v = c.win[1] + (size_t)u * c.W * kD;
      src.ring = true;
      src.row0 = blk * 16;
      src.nvalid = 0;
      src.W = c.W;
      src.first = first;
      src.nwin = nw;
      bool any = false;
#pragma unroll
      for (int r = 0; r < 16; ++r) any |= src.valid(r);
      if (any) process_block(src, st, p.scale_log2, lane);
    }
  }
  const size_t pidx = ((size_t)u * S + split) * kConsumerWarps + warp;
  store_partial(st, p.ws_o, p.ws_ml, pidx, p.G, lane);
}

// ---------------------------------------------------------------- K3: combine partials
__global__ void mstf_combine_kernel(const float* __restrict__ ws_o, const float* __restrict__ ws_ml, int nparts,
                                    int G, void* out, int out_f16) {
  const int u = blockIdx.x;
  const int h = threadIdx.x / kD, ch = threadIdx.x % kD;
  if (h >= G) return;
  float M = -INFINITY;
  for (int i = 0; i < nparts; ++i) M = fmaxf(M, ws_ml[(((size_t)u * nparts + i) * G + h) * 2]);
  float L = 0.f, acc = 0.f;
  for (int i = 0; i < nparts; ++i) {
    const size_t pi = (size_t)u * nparts + i;
    const float m = ws_ml[(pi * G + h) * 2];
    if (m == -INFINITY) continue;
    const float w = exp2f(m - M);
    L += w * ws_ml[(pi * G + h) * 2 + 1];
    acc += w * ws_o[(pi * G + h) * kD + ch];
  }
  const float o = acc / L;
  const size_t oi = ((size_t)u * G + h) * kD + ch;
  if (out_f16)
    reinterpret_cast<__half*>(out)[oi] = __float2half_rn(o);
  else
    reinterpret_cast<float*>(out)[oi] = o;
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
    DenseSrc src;
    src.k = k + (size_t)u * t_max * kD;
    src.v = v + (size_t)u * t_max * kD;
    src.ring = false;
    src.W = src.first = src.nwin = 0;
    src.row0 = b * 16;
    src.nvalid = min(16, n - b * 16);
    process_block(src, st, scale_log2, lane);
  }
  store_partial(st, ws_o, ws_ml, ((size_t)u * S + split) * kConsumerWarps + warp, G, lane);
}

// ---------------------------------------------------------------- host side
int32_t max_splits_for(int32_t U, int32_t capacity) {
  const int32_t chunks = (capacity + kChunk - 1) / kChunk;
  int32_t s = (4 * 148 + U - 1) / U;
  if (s > chunks) s = chunks;
  return s < 1 ? 1 : s;
}

size_t attention_ws_bytes(int32_t U, int32_t G, int32_t max_splits) {
  const size_t parts = (size_t)U * max_splits * kConsumerWarps;
  return parts * G * (kD + 2) * sizeof(float) + 256;
}

AttnPlan plan_attention(int32_t U, int32_t max_comp, int32_t kpad_k, int32_t kpad_v, int32_t sm_count) {
  AttnPlan pl;
  pl.stage_bytes = kChunk * (16 + 2 * kpad_k + 16 + 2 * kpad_v);
  int ns = (96 * 1024) / pl.stage_bytes;
  pl.nstage = ns < 2 ? 2 : (ns > 8 ? 8 : ns);
  const int32_t chunks = (max_comp + kChunk - 1) / kChunk;
  int32_t target = 3 * sm_count;
  int32_t s = (target + U - 1) / U;
  const int32_t cap_s = chunks / 2 > 1 ? chunks / 2 : 1;  // >= 2 chunks per split
  if (s > cap_s) s = cap_s;
  pl.splits = s < 1 ? 1 : s;
  return pl;
}

cudaError_t launch_sparse_attention(const CacheView& c, const AttnPlan& plan, int32_t G, const uint16_t* q,
                                    float scale, void* out, int32_t out_f16, void* ws, cudaStream_t s) {
  AttnParams p;
  p.c = c;
  p.q = q;
  p.G = G;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.nstage = plan.nstage;
  p.stage_bytes = plan.stage_bytes;
  p.off_kval = kChunk * 16;
  p.off_vbm = p.off_kval + kChunk * 2 * c.kpad[0];
  p.off_vval = p.off_vbm + kChunk * 16;
  const size_t parts = (size_t)c.U * plan.splits * kConsumerWarps;
  p.ws_o = reinterpret_cast<float*>(ws);
  p.ws_ml = p.ws_o + parts * G * kD;
  const int smem = kBarBytes + plan.nstage * plan.stage_bytes;
  cudaError_t e = cudaFuncSetAttribute(mstf_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  mstf_attn_kernel<<<dim3(plan.splits, c.U), kThreads, smem, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  mstf_combine_kernel<<<c.U, G * kD, 0, s>>>(p.ws_o, p.ws_ml, plan.splits * kConsumerWarps, G, out, out_f16);
  return cudaGetLastError();
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
  mstf_combine_kernel<<<U, G * kD, 0, s>>>(ws_o, ws_ml, splits * kConsumerWarps, G, out, out_f16);
  return cudaGetLastError();
}

}  // namespace mstf
