// attention.cu -- K2/K3: decode attention directly over the compressed cache
// (Algorithm 1), and the dense-KV baseline on the same skeleton.
//
// Work item = one 16-token block of one unit (compressed records, or rows of the dense
// window ring). Every kernel below runs K/V warp-specialised pairs: K-warp w expands a
// block of K records into mma fragments, computes S^T[16 tok x 8 heads] = K_blk . q^T
// (a5/a6, 8 x mma.m16n8k16, fp32 accumulate), runs the online softmax (a7, exp2 with
// log2e folded into the scale) and hands {P^T fp16 fragments, rescale factors} through a
// 2-slot shared-memory mailbox (mbarriers hfull/hempty) to V-warp w, which expands the
// same block of V records and accumulates O^T[128 ch x 8 heads] += V_blk^T . P^T (a8).
// "Load as compressed, compute as dense": the expansion writes zeros at pruned
// channels in registers; nothing dense ever touches HBM.
//
// Expansion ("gather"): a warp writes each token's packed values into a shifted pair
// array Y[m] = (h[m-1], h[m]) in shared memory; channel pair (2j, 2j+1) of bitmap word w
// is then ONE 32-bit load at Y[popc(w & bits <= 2j)] masked by the two bitmap bits
// (prmt sign-replicate masks), so a lane builds its fragments without branches.
//
// Kernels
//   mstf_attn_reg_kernel<NK,NV>   (k_pad 16/32/40/64: the 70% and 50% sparsity paths) 8 warps, each
//       warp streams its blocks' records straight into registers with a one-block
//       software pipeline, builds the pair arrays from registers, gathers, mma. Work
//       schedule: stream-K (units' blocks concatenated, equal ranges over one wave of
//       2 CTAs per SM; see UnitSched below) or split grid (S, U). The last CTA to finish
//       a unit merges its partials (a9) in the same launch.
//   mstf_attn_kv_kernel<NK,NV,I>  (other k_pad, or K != V sparsity) 8 consumer warps +
//       1 producer warp streaming 64-token chunks (K bitmaps, K values, V bitmaps,
//       V values: four cp.async.bulk copies) into an mbarrier-guarded smem ring; split grid.
//   mstf_combine_kernel           merges the kv kernel's split partials (a9).
//   mstf_dense_attn_kernel        dense-KV baseline (same mma/softmax code, no expansion).
//
// Fragment <-> channel mapping (free permutations of the contraction / output index):
//   K mma, lane (g = lane/4, t = lane%4): tokens g and g+8, channels 32t..32t+31
//     (= bitmap word t of the token); k-step s uses channels 32t+4s+{0,1} (a0/a1, b0)
//     and 32t+4s+{2,3} (a2/a3, b1).
//   V mma, m-tile i: row r <-> channel 8r+i, i.e. lane (g,t) expands bitmap bytes g and
//     g+8 of tokens 2t, 2t+1, 2t+8, 2t+9.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "compress_dev.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace mstf {


struct AttnParams {
  CacheView c;
  const uint16_t* q;  // [U][G][kD]
  float* ws_o;        // [U][S][NW][G][kD]
  float* ws_ml;       // [U][S][NW][G][2]
  int G;
  float scale_log2;
  int nstage, stage_bytes;
  int off_kval, off_vbm, off_vval;  // byte offsets inside a stage (kbm at 0)
  uint32_t off_pairs;               // byte offset of the per-warp pair-array regions
  uint32_t off_handoff;             // byte offset of the K->V mailbox (split kernel)
  uint32_t reg_k, reg_v;            // per-warp pair-array region bytes (K, V)
  int* tickets;                     // [U] arrival counters for the fused combine
  int32_t sk;                       // 1: register kernel, stream-K schedule; 0: split grid (S, U)
  int32_t sk_nb;                    // stream-K: items per unit if uniform, 0 = ragged (smem prefix)
  uint32_t off_pref;                // stream-K ragged: byte offset of the prefix array in smem
  int32_t trace;                    // dev: record per-CTA start/end/SM into g_trace
  int32_t sk_static;                // stream-K: cost units split statically (worker P: [B(P), B(P+1)))
  int32_t sk_c;                     // stream-K: items per dynamic tail chunk
  int32_t sk_nchunks;               // stream-K: dynamic tail chunks (0 = static only)
  int32_t sk_total;                 // stream-K: total items
  int* sk_ctr;                      // stream-K: [0] next tail chunk, [1] workers done (zero between calls)
  int32_t sk_np;                    // stream-K: workers (warp pairs) = 4 * grid
  int32_t sk_cs, sk_cw;             // stream-K cost model: per-unit start cost, cost per window block
  // fused decode step (append + attention in one launch; uniform caches): counters before
  // (nc_old, nw_old) and after (unc, unw) the append, whether a window token was evicted into
  // record nc_old, the new tokens, and per-unit ready flags [2U] stamped with `epoch`
  int32_t fuse, evict, nc_old, nw_old, unc, unw, epoch;
  const uint16_t* k_new;
  const uint16_t* v_new;
  int* ready;
  int* sk_pref;                     // stream-K ragged: per-unit item prefix in the workspace (U+1)
  void* out;
  int out_f16;
  float* part_ml;  // non-null: write the softmax partials (m, l) [U][G][2] and o [U][G][kD] instead of O
  float* part_o;
};

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

// Mask for dibit j of word w (channels 2j, 2j+1 -> halves lo, hi): 0xFFFF where the
// channel is kept. cp[s] = w << (7 - s) puts bit 8m+s at the sign bit of byte m;
// prmt's sign-replicate mode turns the two needed sign bits into byte masks.
template <int J>
__device__ __forceinline__ uint32_t dibit_mask(const uint32_t (&cp)[8]) {
  constexpr int m = J / 4, s0 = 2 * (J % 4);
  constexpr uint32_t lo = 8 | m, hi = 8 | (4 + m);
  constexpr uint32_t sel = lo | (lo << 4) | (hi << 8) | (hi << 12);
  return prmt(cp[s0], cp[s0 + 1], sel);
}

__device__ __forceinline__ void shifted_copies(uint32_t w, uint32_t (&cp)[8]) {
#pragma unroll
  for (int s = 0; s < 8; ++s) cp[s] = w * (1u << (7 - s));
}

// Per-block register operands, already expanded (zeros at pruned channels):
//   k[r][j] : token g (r=0) / g+8 (r=1), channels 32t+2j, 32t+2j+1   (K mma A operand)
//   v[x][j] : token {2t, 2t+1, 2t+8, 2t+9}[x], channels 16g+2j, 16g+2j+1 (V mma A operand)
struct BlockRegs {
  uint32_t k[2][16];
  uint32_t v[4][8];
};

// ---------------------------------------------------------------- compressed source
// Shifted pair array of one token: Y[m] = (h[m-1], h[m]) (h[-1] = 0), m = 0..kpad, in shared
// memory, so the pair of values a dibit needs is ONE aligned 32-bit load: for dibit j of a
// word with exclusive token prefix P, Y[P + popc(word & bits<=2j)] holds (value of channel
// 2j if kept else previous, value of channel 2j+1 if kept); the mask zeroes pruned halves.
struct CompBlock {
  const uint8_t* smem;   // dynamic smem base (generic)
  uint32_t kbm, kval, vbm, vval;  // byte offsets of this stage's arrays
  uint32_t yk, yv;       // byte offsets of this warp's pair-array regions
  int kpk, kpv, tok0, nvalid;
  uint32_t strk, strv;   // pair-array stride per token (bytes)
};

// Materialise a value in one register (stops the compiler from re-associating base + stride * pc
// into several adds per gather).
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
  asm("mov.b32 %0, %0;" : "+r"(x));
  return x;
}
// 32-bit shared-window loads / stores (absolute shared addresses, no generic->shared conversion).
__device__ __forceinline__ uint32_t lds_abs(uint32_t saddr) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr) : "memory");
  return v;
}
// Gather only when the dibit keeps a channel (mask != 0): idle lanes take no bank slot.
__device__ __forceinline__ uint32_t lds_abs_masked(uint32_t saddr, uint32_t mask) {
  uint32_t v = 0;
  asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.shared.u32 %0, [%1];\n\t}"
      : "+r"(v) : "r"(saddr), "r"(mask) : "memory");
  return v & mask;
}
__device__ __forceinline__ void sts_abs(uint32_t saddr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_s32(const uint8_t* smem, uint32_t off) {
  return *reinterpret_cast<const uint32_t*>(smem + off);
}

// Build the warp's 16 pair arrays of one tensor from the raw packed values of the stage.
template <int NCH>  // chunks of 8 values per token (kpad / 8); 0 = runtime
__device__ __forceinline__ void build_pairs(uint8_t* smem, uint32_t raw, uint32_t y, int kp_rt, uint32_t stride,
                                            int tok0, int lane) {
  const int nch = NCH ? NCH : (kp_rt >> 3);
  const int kp = 8 * nch;
#pragma unroll
  for (int cid = lane; cid < 16 * nch; cid += 32) {
    const int tau = cid / nch, c = cid - tau * nch;
    const uint32_t src = raw + (uint32_t)((tok0 + tau) * kp * 2 + 16 * c);
    const uint4 a = *reinterpret_cast<const uint4*>(smem + src);
    const uint32_t nxt = (c + 1 < nch) ? ld_s32(smem, src + 16) : 0u;
    const uint32_t ybase = y + (uint32_t)tau * stride + 12;  // Y[m] at ybase + 4m
    uint4 lo, hi;
    lo.x = a.x; lo.y = prmt(a.x, a.y, 0x5432); lo.z = a.y; lo.w = prmt(a.y, a.z, 0x5432);
    hi.x = a.z; hi.y = prmt(a.z, a.w, 0x5432); hi.z = a.w; hi.w = prmt(a.w, nxt, 0x5432);
    *reinterpret_cast<uint4*>(smem + ybase + 4 * (8 * c + 1)) = lo;
    *reinterpret_cast<uint4*>(smem + ybase + 4 * (8 * c + 5)) = hi;
    if (c == 0) *reinterpret_cast<uint32_t*>(smem + ybase) = a.x << 16;
  }
}

// Expand the 16 dibits of word w (token prefix folded into `base`) into out[16].
__device__ __forceinline__ void gather_word16(const uint8_t* smem, uint32_t w, uint32_t base, uint32_t (&out)[16]) {
  uint32_t cp[8];
  shifted_copies(w, cp);
#define MSTF_G(J)                                                                 \
  {                                                                               \
    const uint32_t pc = __popc(w * (1u << (31 - 2 * J)));                         \
    out[J] = ld_s32(smem, base + 4u * pc) & dibit_mask<J>(cp);                    \
  }
  MSTF_G(0) MSTF_G(1) MSTF_G(2) MSTF_G(3) MSTF_G(4) MSTF_G(5) MSTF_G(6) MSTF_G(7)
  MSTF_G(8) MSTF_G(9) MSTF_G(10) MSTF_G(11) MSTF_G(12) MSTF_G(13) MSTF_G(14) MSTF_G(15)
#undef MSTF_G
}
// Expand 8 dibits (bits 0..15 of hw) into out[8].
__device__ __forceinline__ void gather_half8(const uint8_t* smem, uint32_t hw, uint32_t base, uint32_t (&out)[8]) {
  uint32_t cp[8];
  shifted_copies(hw, cp);
#define MSTF_G(J)                                                                 \
  {                                                                               \
    const uint32_t pc = __popc(hw * (1u << (31 - 2 * J)));                        \
    out[J] = ld_s32(smem, base + 4u * pc) & dibit_mask<J>(cp);                    \
  }
  MSTF_G(0) MSTF_G(1) MSTF_G(2) MSTF_G(3) MSTF_G(4) MSTF_G(5) MSTF_G(6) MSTF_G(7)
#undef MSTF_G
}

// K half: pair arrays of the 16 K tokens, then the K operand (k[2][16]).
template <int NK>
__device__ __forceinline__ void fill_k(const CompBlock& cb, uint8_t* smem, uint32_t (&kr)[2][16], int lane) {
  const int g = lane >> 2, t = lane & 3;
  build_pairs<NK>(smem, cb.kval, cb.yk, cb.kpk, cb.strk, cb.tok0, lane);
  const uint32_t kw0 = g < cb.nvalid ? ld_s32(smem, cb.kbm + 16 * (cb.tok0 + g) + 4 * t) : 0u;
  const uint32_t kw1 = g + 8 < cb.nvalid ? ld_s32(smem, cb.kbm + 16 * (cb.tok0 + g + 8) + 4 * t) : 0u;
  const uint32_t pk = __popc(kw0) | (__popc(kw1) << 16);
  uint32_t ik = pk;
#pragma unroll
  for (int o = 1; o < 4; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, ik, o, 4);
    if (t >= o) ik += y;
  }
  const uint32_t ek = ik - pk;
  __syncwarp();
  const uint32_t bk0 = cb.yk + (uint32_t)g * cb.strk + 12 + 4 * (ek & 0xFFFF);
  const uint32_t bk1 = bk0 + 8 * cb.strk + 4 * ((ek >> 16) - (ek & 0xFFFF));
  gather_word16(smem, kw0, bk0, kr[0]);
  gather_word16(smem, kw1, bk1, kr[1]);
}

// V half: pair arrays of the 16 V tokens, then the V operand (v[4][8]).
template <int NV>
__device__ __forceinline__ void fill_v(const CompBlock& cb, uint8_t* smem, uint32_t (&vr)[4][8], int lane) {
  const int g = lane >> 2, t = lane & 3;
  build_pairs<NV>(smem, cb.vval, cb.yv, cb.kpv, cb.strv, cb.tok0, lane);
  const uint32_t vw0 = g < cb.nvalid ? ld_s32(smem, cb.vbm + 16 * (cb.tok0 + g) + 4 * t) : 0u;
  const uint32_t vw1 = g + 8 < cb.nvalid ? ld_s32(smem, cb.vbm + 16 * (cb.tok0 + g + 8) + 4 * t) : 0u;
  const uint32_t pv = __popc(vw0) | (__popc(vw1) << 16);
  uint32_t iv = pv;
#pragma unroll
  for (int o = 1; o < 4; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, iv, o, 4);
    if (t >= o) iv += y;
  }
  const uint32_t ev = iv - pv;
  __syncwarp();
  const int sa = 8 * t + (g >> 1), sb = sa + 4, hsh = 16 * (g & 1);
  const uint32_t w2t = __shfl_sync(0xffffffffu, vw0, sa), w2t8 = __shfl_sync(0xffffffffu, vw1, sa);
  const uint32_t w2t1 = __shfl_sync(0xffffffffu, vw0, sb), w2t9 = __shfl_sync(0xffffffffu, vw1, sb);
  const uint32_t pa = __shfl_sync(0xffffffffu, ev, sa), pb = __shfl_sync(0xffffffffu, ev, sb);
  const uint32_t ws[4] = {w2t, w2t1, w2t8, w2t9};
  const uint32_t ps[4] = {pa & 0xFFFF, pb & 0xFFFF, pa >> 16, pb >> 16};
  const int tk[4] = {2 * t, 2 * t + 1, 2 * t + 8, 2 * t + 9};
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const uint32_t extra = (g & 1) ? __popc(ws[x] & 0xFFFFu) : 0u;
    const uint32_t base = cb.yv + (uint32_t)tk[x] * cb.strv + 12 + 4 * (ps[x] + extra);
    gather_half8(smem, ws[x] >> hsh, base, vr[x]);
  }
}

// ---------------------------------------------------------------- interleaved pair arrays (v3)
// Thread-per-token build: lane L handles token tau = L >> 1, half h = L & 1 of one tensor's 16
// tokens. With kp = kpad, half h writes entries m = M0(h) + e, e = 0..E-1, E = kp/2 + 2,
// M0(1) = kp/2 + 2 (entries past kp are padding rows). Y[m] = (h[m-1], h[m]).
// Layouts (word offsets inside a warp region; 32-bit entries):
//   K : region K_{tau>>3}, word 8*m + (tau & 7)        -> a K gather row touches 8 tokens in
//       distinct banks; regions K0/K1 sit 8 banks apart so the build stores are conflict-free
//   V : region V_r, r = (tau & 1) + 2*(tau >> 3), word 4*m + ((tau >> 1) & 3)
//       -> a V gather touches 4 tokens x 8 lanes; region bank offsets {0, 4, 16, 20}.
template <int NCH>
struct PairGeom {
  static constexpr int kp = 8 * NCH;
  static constexpr int E = kp / 2 + 2;   // entries per half-lane
  static constexpr int rows = kp + 4;    // rows per region (>= M0(1) + E)
  static constexpr int nw = E / 2 + 1;   // raw words loaded per half-lane
};

// Region word offsets, padded so that region bases have the required bank offsets.
__host__ __device__ constexpr int pad_to_bank(int off, int bank) {
  return off + ((bank - (off & 31)) & 31);
}
template <int NCH>
struct KLayout {
  static constexpr int rows = PairGeom<NCH>::rows;
  static constexpr int k0 = 0;
  static constexpr int k1 = pad_to_bank(k0 + 8 * rows, 8);
  static constexpr int words = k1 + 8 * rows;
};
template <int NCH>
struct VLayout {
  static constexpr int rows = PairGeom<NCH>::rows;
  static constexpr int v0 = 0;
  static constexpr int v1 = pad_to_bank(v0 + 4 * rows, 4);
  static constexpr int v2 = pad_to_bank(v1 + 4 * rows, 16);
  static constexpr int v3 = pad_to_bank(v2 + 4 * rows, 20);
  static constexpr int words = v3 + 4 * rows;
  __host__ __device__ static constexpr int region(int r) { return r == 0 ? v0 : r == 1 ? v1 : r == 2 ? v2 : v3; }
};

template <int NCH, bool IS_V>
__device__ __forceinline__ void build_interleaved(uint8_t* smem, uint32_t raw, uint32_t ybase, int tok0, int lane) {
  using Gm = PairGeom<NCH>;
  const int tau = lane >> 1, h = lane & 1;
  const int m0 = h ? Gm::kp / 2 + 2 : 0;
  // raw words wb .. wb + nw - 1 of token tau, wb = m0/2 - 1 (word -1 == 0)
  const uint32_t src = raw + (uint32_t)((tok0 + tau) * Gm::kp * 2) + 4u * (uint32_t)(m0 / 2 - 1);
  uint32_t W[Gm::nw];
  W[0] = h ? ld_s32(smem, src) : 0u;
#pragma unroll
  for (int i = 1; i < Gm::nw; ++i) W[i] = ld_s32(smem, src + 4 * i);
  uint32_t dst, step;
  if (IS_V) {
    const int r = (tau & 1) + 2 * (tau >> 3);
    dst = ybase + 4u * (uint32_t)(VLayout<NCH>::region(r) + ((tau >> 1) & 3) + 4 * m0);
    step = 16;
  } else {
    dst = ybase + 4u * (uint32_t)((tau >> 3 ? KLayout<NCH>::k1 : KLayout<NCH>::k0) + (tau & 7) + 8 * m0);
    step = 32;
  }
#pragma unroll
  for (int e = 0; e < Gm::E; ++e) {
    const uint32_t y = (e & 1) ? W[(e + 1) >> 1] : prmt(W[e >> 1], W[(e >> 1) + 1], 0x5432);
    *reinterpret_cast<uint32_t*>(smem + dst + step * e) = y;
  }
}

// Expand 16 dibits of word w; entry r of this token's pair array at base + stride * r.
template <int STRIDE>
__device__ __forceinline__ void gather16_s(const uint8_t* smem, uint32_t w, uint32_t base_in, uint32_t (&out)[16]) {
  const uint32_t base = opaque(base_in + smem_u32(smem));
  uint32_t cp[8];
  shifted_copies(w, cp);
#define MSTF_G(J)                                                                 \
  {                                                                               \
    const uint32_t pc = __popc(w * (1u << (31 - 2 * J)));                         \
    out[J] = lds_abs_masked(base + STRIDE * pc, dibit_mask<J>(cp));                \
  }
  MSTF_G(0) MSTF_G(1) MSTF_G(2) MSTF_G(3) MSTF_G(4) MSTF_G(5) MSTF_G(6) MSTF_G(7)
  MSTF_G(8) MSTF_G(9) MSTF_G(10) MSTF_G(11) MSTF_G(12) MSTF_G(13) MSTF_G(14) MSTF_G(15)
#undef MSTF_G
}
template <int STRIDE>
__device__ __forceinline__ void gather8_s(const uint8_t* smem, uint32_t hw, uint32_t base_in, uint32_t (&out)[8]) {
  const uint32_t base = opaque(base_in + smem_u32(smem));
  uint32_t cp[8];
  shifted_copies(hw, cp);
#define MSTF_G(J)                                                                 \
  {                                                                               \
    const uint32_t pc = __popc(hw * (1u << (31 - 2 * J)));                        \
    out[J] = lds_abs_masked(base + STRIDE * pc, dibit_mask<J>(cp));                \
  }
  MSTF_G(0) MSTF_G(1) MSTF_G(2) MSTF_G(3) MSTF_G(4) MSTF_G(5) MSTF_G(6) MSTF_G(7)
#undef MSTF_G
}

// Interleaved V gather (register-staged kernel): the two lanes that share a bitmap word take
// alternating dibits rather than its two 16-bit halves, so in one gather instruction they read
// adjacent pair-array rows (fewer shared-memory bank conflicts; same instruction count).
// V: the lane pair (2w', 2w'+1) of a token shares bitmap word wv; lane parity h takes its
// dibits 2i + h (channels 32w' + 4i + 2h, +1), i = 0..7. base = absolute smem address of pair
// entry (kept values before word wv).
template <int STRIDE>
__device__ __forceinline__ void gather8_il(uint32_t wv, uint32_t base, int h, uint32_t (&out)[8]) {
  // bits p = 4i + 2h, p + 1 sit in byte i/2 at bit 4(i&1) + 2h. One lane-dependent shift
  // (wp = wv << (2 - 2h)); every other shift is by an immediate, so it can issue on the FMA pipe
  // (IMAD.SHL) instead of the busier ALU pipe. Dropping wv's top bits for h = 0 is harmless: no
  // shift below needs bits above 28 + 2h.
  const uint32_t wp = wv << (2 - 2 * h);
  const uint32_t ce0 = wp * (1u << 5), ce1 = wp * (1u << 4);  // i even: wv << (7 - 2h), << (6 - 2h)
  const uint32_t co0 = wp * 2u, co1 = wp;                      // i odd:  wv << (3 - 2h), << (2 - 2h)
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t m = i >> 1;
    const uint32_t sel = (8u | m) | ((8u | m) << 4) | ((12u | m) << 8) | ((12u | m) << 12);
    const uint32_t pc = __popc(wp * (1u << (29 - 4 * i)));  // kept channels <= 4i + 2h
    out[i] = lds_abs_masked(base + STRIDE * pc, (i & 1) ? prmt(co0, co1, sel) : prmt(ce0, ce1, sel));
  }
}

template <int NK>
__device__ __forceinline__ void fill_k3(const CompBlock& cb, uint8_t* smem, uint32_t (&kr)[2][16], int lane) {
  const int g = lane >> 2, t = lane & 3;
  build_interleaved<NK, false>(smem, cb.kval, cb.yk, cb.tok0, lane);
  const uint32_t kw0 = g < cb.nvalid ? ld_s32(smem, cb.kbm + 16 * (cb.tok0 + g) + 4 * t) : 0u;
  const uint32_t kw1 = g + 8 < cb.nvalid ? ld_s32(smem, cb.kbm + 16 * (cb.tok0 + g + 8) + 4 * t) : 0u;
  const uint32_t pk = __popc(kw0) | (__popc(kw1) << 16);
  uint32_t ik = pk;
#pragma unroll
  for (int o = 1; o < 4; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, ik, o, 4);
    if (t >= o) ik += y;
  }
  const uint32_t ek = ik - pk;
  __syncwarp();
  const uint32_t b0 = cb.yk + 4u * (uint32_t)(KLayout<NK>::k0 + g) + 32u * (ek & 0xFFFF);
  const uint32_t b1 = cb.yk + 4u * (uint32_t)(KLayout<NK>::k1 + g) + 32u * (ek >> 16);
  gather16_s<32>(smem, kw0, b0, kr[0]);
  gather16_s<32>(smem, kw1, b1, kr[1]);
}

template <int NV>
__device__ __forceinline__ void fill_v3(const CompBlock& cb, uint8_t* smem, uint32_t (&vr)[4][8], int lane) {
  const int g = lane >> 2, t = lane & 3;
  build_interleaved<NV, true>(smem, cb.vval, cb.yv, cb.tok0, lane);
  const uint32_t vw0 = g < cb.nvalid ? ld_s32(smem, cb.vbm + 16 * (cb.tok0 + g) + 4 * t) : 0u;
  const uint32_t vw1 = g + 8 < cb.nvalid ? ld_s32(smem, cb.vbm + 16 * (cb.tok0 + g + 8) + 4 * t) : 0u;
  const uint32_t pv = __popc(vw0) | (__popc(vw1) << 16);
  uint32_t iv = pv;
#pragma unroll
  for (int o = 1; o < 4; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, iv, o, 4);
    if (t >= o) iv += y;
  }
  const uint32_t ev = iv - pv;
  __syncwarp();
  const int sa = 8 * t + (g >> 1), sb = sa + 4, hsh = 16 * (g & 1);
  const uint32_t w2t = __shfl_sync(0xffffffffu, vw0, sa), w2t8 = __shfl_sync(0xffffffffu, vw1, sa);
  const uint32_t w2t1 = __shfl_sync(0xffffffffu, vw0, sb), w2t9 = __shfl_sync(0xffffffffu, vw1, sb);
  const uint32_t pa = __shfl_sync(0xffffffffu, ev, sa), pb = __shfl_sync(0xffffffffu, ev, sb);
  const uint32_t ws[4] = {w2t, w2t1, w2t8, w2t9};
  const uint32_t ps[4] = {pa & 0xFFFF, pb & 0xFFFF, pa >> 16, pb >> 16};
  // token 2t+c: region r = (c & 1) + 2 * (c >> 3) = x for x = 0..3 (c = 0, 1, 8, 9), slot t
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const uint32_t extra = (g & 1) ? __popc(ws[x] & 0xFFFFu) : 0u;
    const uint32_t base = cb.yv + 4u * (uint32_t)(VLayout<NV>::region(x) + t) + 16u * (ps[x] + extra);
    gather8_s<16>(smem, ws[x] >> hsh, base, vr[x]);
  }
}

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
// {P^T fragment kappa 0, kappa 1, alpha head 2t, alpha head 2t+1}.
struct KState {
  float m0, m1, l0, l1;
  uint32_t qf[16];
};
__device__ __forceinline__ uint4 k_block(const uint32_t (&kr)[2][16], bool vg, bool vg8, KState& st, float scale_log2) {
  float sc[4] = {0.f, 0.f, 0.f, 0.f}, sd[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int s = 0; s < 8; s += 2) {
    mma16816(sc, kr[0][2 * s], kr[1][2 * s], kr[0][2 * s + 1], kr[1][2 * s + 1], st.qf[2 * s], st.qf[2 * s + 1]);
    mma16816(sd, kr[0][2 * s + 2], kr[1][2 * s + 2], kr[0][2 * s + 3], kr[1][2 * s + 3], st.qf[2 * s + 2],
             st.qf[2 * s + 3]);
  }
  const float x0 = vg ? (sc[0] + sd[0]) * scale_log2 : -INFINITY;
  const float x1 = vg ? (sc[1] + sd[1]) * scale_log2 : -INFINITY;
  const float x2 = vg8 ? (sc[2] + sd[2]) * scale_log2 : -INFINITY;
  const float x3 = vg8 ? (sc[3] + sd[3]) * scale_log2 : -INFINITY;
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
  return make_uint4(movmatrix_t(pack_half2(p0, p1)), movmatrix_t(pack_half2(p2, p3)), __float_as_uint(a0),
                    __float_as_uint(a1));
}

// V-warp block step: rescale, then O^T += V-pairs . P (even / odd channel MMAs).
__device__ __forceinline__ void v_block(const uint32_t (&vr)[4][8], const uint4 h, float (&acc)[2][4][4]) {
  const float a0 = __uint_as_float(h.z), a1 = __uint_as_float(h.w);
  if (__any_sync(0xffffffffu, a0 != 1.f || a1 != 1.f)) {
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[e][i][0] *= a0; acc[e][i][1] *= a1; acc[e][i][2] *= a0; acc[e][i][3] *= a1;
      }
  }
  const uint32_t m[2] = {h.x, h.y};
#pragma unroll
  for (int kap = 0; kap < 2; ++kap) {
    const uint32_t be0 = m[kap] & 0xFFFFu, be1 = m[kap] >> 16, bo0 = m[kap] << 16, bo1 = m[kap] & 0xFFFF0000u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t a0r = vr[2 * kap][i], a1r = vr[2 * kap][4 + i];
      const uint32_t a2r = vr[2 * kap + 1][i], a3r = vr[2 * kap + 1][4 + i];
      mma16816(acc[0][i], a0r, a1r, a2r, a3r, be0, be1);
      mma16816(acc[1][i], a0r, a1r, a2r, a3r, bo0, bo1);
    }
  }
}

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
// memory mailbox (mbarriers hfull / hempty); the V-warp gathers V and accumulates P.V.
constexpr int kKVWarps = 8;
constexpr int kThreadsKV = (kKVWarps + 1) * 32;
constexpr int kBarBytesKV = 256;   // full[8], empty[8], hfull[8], hempty[8]
constexpr int kHandoffBytes = 4 * 2 * 32 * 16;
constexpr int kBarBytesReg = 256;  // register kernel: hfull, hempty, dfull, dempty [4 pairs][2]

template <int NK, int NV, bool INTERLEAVED>
__global__ void __launch_bounds__(kThreadsKV, 2) mstf_attn_kv_kernel(const AttnParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 8;
  uint64_t* hfull = full + 16;
  uint64_t* hempty = full + 24;
  uint4* handoff = reinterpret_cast<uint4*>(smem + p.off_handoff);

  const int u = blockIdx.y, split = blockIdx.x, S = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const CacheView& c = p.c;
  pdl_launch_dependents();
  pdl_wait();  // cache, counters and q may be written by the previous kernel in the stream
  const int n = c.n_comp[u];
  const int chunks_total = (n + kChunk - 1) / kChunk;
  const int cps = (chunks_total + S - 1) / S;
  const int cbeg = min(split * cps, chunks_total), cend = min(cbeg + cps, chunks_total);
  const int nchunks = cend - cbeg;

  if (threadIdx.x == 0) {
    for (int i = 0; i < p.nstage; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kKVWarps);
    }
    for (int i = 0; i < 8; ++i) {
      mbar_init(&hfull[i], 1);
      mbar_init(&hempty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kKVWarps) {
    // ---------------- producer (same as the fused kernel)
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
        uint8_t* sb = smem + kBarBytesKV + (size_t)st * p.stage_bytes;
        mbar_arrive_expect_tx(&full[st], 2 * bbm + bk + bv);
        bulk_g2s(sb, kbm + (size_t)tok0 * 16, bbm, &full[st]);
        bulk_g2s(sb + p.off_kval, kval + (size_t)tok0 * 2 * kpk, bk, &full[st]);
        bulk_g2s(sb + p.off_vbm, vbm + (size_t)tok0 * 16, bbm, &full[st]);
        bulk_g2s(sb + p.off_vval, vval + (size_t)tok0 * 2 * kpv, bv, &full[st]);
      }
    }
    return;
  }

  const bool is_k = warp < 4;
  const int w = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  CompBlock cb;
  cb.smem = smem;
  cb.kpk = c.kpad[0];
  cb.kpv = c.kpad[1];
  cb.strk = 4 * cb.kpk + 16;
  cb.strv = 4 * cb.kpv + 16;
  cb.yk = p.off_pairs + (uint32_t)w * p.reg_k;
  cb.yv = p.off_pairs + 4 * p.reg_k + (uint32_t)w * p.reg_v;
  cb.tok0 = 16 * w;
  const size_t pidx = ((size_t)u * S + split) * kConsumerWarps + w;
  const int nwin_blocks = (split == S - 1 && c.W > 0) ? (c.W + 15) / 16 : 0;
  const int nw = c.n_win[u];
  const int first = c.W > 0 ? n % c.W : 0;

  if (is_k) {
    // ================= K-warp
    KState st;
    st.m0 = st.m1 = -INFINITY;
    st.l0 = st.l1 = 0.f;
    if (g < p.G) {
      const uint4* qp = reinterpret_cast<const uint4*>(p.q + ((size_t)u * p.G + g) * kD + 32 * t);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 x = qp[i];
        st.qf[4 * i] = x.x; st.qf[4 * i + 1] = x.y; st.qf[4 * i + 2] = x.z; st.qf[4 * i + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) st.qf[i] = 0;
    }
    int blk = 0;
    auto handoff_put = [&](const uint4 h) {
      const int slot = blk & 1;
      if (blk >= 2) mbar_wait(&hempty[2 * w + slot], ((blk >> 1) - 1) & 1);
      handoff[(w * 2 + slot) * 32 + lane] = h;
      __syncwarp();
      if (lane == 0) mbar_arrive(&hfull[2 * w + slot]);
      ++blk;
    };
    for (int i = 0; i < nchunks; ++i) {
      const int sidx = i % p.nstage;
      mbar_wait(&full[sidx], (i / p.nstage) & 1);
      const uint32_t sb = kBarBytesKV + (uint32_t)sidx * p.stage_bytes;
      const int nvalid = min(16, n - (cbeg + i) * kChunk - 16 * w);
      uint32_t kr[2][16];
      if (nvalid > 0) {
        cb.kbm = sb;
        cb.kval = sb + p.off_kval;
        cb.nvalid = nvalid;
        if constexpr (INTERLEAVED && NK > 0) fill_k3<NK>(cb, smem, kr, lane); else fill_k<NK>(cb, smem, kr, lane);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sidx]);
      if (nvalid > 0) handoff_put(k_block(kr, g < nvalid, g + 8 < nvalid, st, p.scale_log2));
    }
    for (int blkw = w; blkw < nwin_blocks; blkw += 4) {
      DenseBlock db;
      db.k = c.win[0] + (size_t)u * c.W * kD;
      db.v = c.win[1] + (size_t)u * c.W * kD;
      db.ring = true; db.row0 = blkw * 16; db.nvalid = 0; db.W = c.W; db.first = first; db.nwin = nw;
      bool any = false;
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) any |= db.valid(rr);
      if (!any) continue;
      uint32_t kr[2][16];
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int tok = g + 8 * x;
        if (db.valid(tok)) {
          const uint4* pp = reinterpret_cast<const uint4*>(db.k + (size_t)(db.row0 + tok) * kD + 32 * t);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 a = pp[j];
            kr[x][4 * j] = a.x; kr[x][4 * j + 1] = a.y; kr[x][4 * j + 2] = a.z; kr[x][4 * j + 3] = a.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) kr[x][j] = 0;
        }
      }
      handoff_put(k_block(kr, db.valid(g), db.valid(g + 8), st, p.scale_log2));
    }
    // partial (m, l)
    float l0 = st.l0, l1 = st.l1;
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, o);
      l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    float* ml = p.ws_ml + pidx * p.G * 2;
    if (g == 0) {
      if (2 * t < p.G) { ml[4 * t] = st.m0; ml[4 * t + 1] = l0; }
      if (2 * t + 1 < p.G) { ml[4 * t + 2] = st.m1; ml[4 * t + 3] = l1; }
    }
  } else {
    // ================= V-warp
    float acc[2][4][4];
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[e][i][0] = acc[e][i][1] = acc[e][i][2] = acc[e][i][3] = 0.f;
    int blk = 0;
    auto handoff_get = [&]() -> uint4 {
      const int slot = blk & 1;
      mbar_wait(&hfull[2 * w + slot], (blk >> 1) & 1);
      const uint4 h = handoff[(w * 2 + slot) * 32 + lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&hempty[2 * w + slot]);
      ++blk;
      return h;
    };
    for (int i = 0; i < nchunks; ++i) {
      const int sidx = i % p.nstage;
      mbar_wait(&full[sidx], (i / p.nstage) & 1);
      const uint32_t sb = kBarBytesKV + (uint32_t)sidx * p.stage_bytes;
      const int nvalid = min(16, n - (cbeg + i) * kChunk - 16 * w);
      uint32_t vr[4][8];
      if (nvalid > 0) {
        cb.vbm = sb + p.off_vbm;
        cb.vval = sb + p.off_vval;
        cb.nvalid = nvalid;
        if constexpr (INTERLEAVED && NV > 0) fill_v3<NV>(cb, smem, vr, lane); else fill_v<NV>(cb, smem, vr, lane);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sidx]);
      if (nvalid > 0) v_block(vr, handoff_get(), acc);
    }
    for (int blkw = w; blkw < nwin_blocks; blkw += 4) {
      DenseBlock db;
      db.k = c.win[0] + (size_t)u * c.W * kD;
      db.v = c.win[1] + (size_t)u * c.W * kD;
      db.ring = true; db.row0 = blkw * 16; db.nvalid = 0; db.W = c.W; db.first = first; db.nwin = nw;
      bool any = false;
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) any |= db.valid(rr);
      if (!any) continue;
      uint32_t vr[4][8];
      const int tk[4] = {2 * t, 2 * t + 1, 2 * t + 8, 2 * t + 9};
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        if (db.valid(tk[x])) {
          const uint4* pp = reinterpret_cast<const uint4*>(db.v + (size_t)(db.row0 + tk[x]) * kD + 16 * g);
          const uint4 a = pp[0], b = pp[1];
          vr[x][0] = a.x; vr[x][1] = a.y; vr[x][2] = a.z; vr[x][3] = a.w;
          vr[x][4] = b.x; vr[x][5] = b.y; vr[x][6] = b.z; vr[x][7] = b.w;
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) vr[x][j] = 0;
        }
      }
      v_block(vr, handoff_get(), acc);
    }
    float* o = p.ws_o + pidx * p.G * kD;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int h = 2 * t + hh;
      if (h < p.G) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          *reinterpret_cast<float2*>(o + h * kD + 16 * g + 2 * i) = make_float2(acc[0][i][hh], acc[1][i][hh]);
          *reinterpret_cast<float2*>(o + h * kD + 16 * g + 8 + 2 * i) =
              make_float2(acc[0][i][2 + hh], acc[1][i][2 + hh]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------- fused split combine (a9)
// Called by every thread of a CTA after its warps stored their partials. The last CTA of the unit
// (ticket counter in the workspace) merges the S * 4 partials and writes the output; the ticket
// is reset to 0 so the workspace is reusable (it must be zeroed once before first use).

// Fused split combine: unit u's partials are [part_begin, part_begin + nparts) and `expected`
// CTAs arrive; the last one to take a ticket merges them. Called by every thread of the CTA.
// Partial slots of unit u: [b1, b1 + n1) and [b2, b2 + n2); each slot holds kConsumerWarps
// per-warp partials; n1 + n2 CTAs arrive.
struct PartRanges {
  int b1, n1, b2, n2;
};

// ---------------------------------------------------------------- K2 v4: register-staged (no TMA ring)
// 4 K-warps + 4 V-warps per CTA; K-warp w and V-warp w+4 own the 16-token blocks
// b = w, w+4, w+8, ... of the split. Each warp loads its tensor's packed values and bitmap
// words for the NEXT block with 64/32-bit global loads into registers (software pipelining),
// then builds the interleaved pair arrays from registers (no shared-memory staging reads).
template <int NCH>
struct RawRegs {
  static constexpr int nw = PairGeom<NCH>::nw;
  uint32_t W[nw];
  uint32_t bm0, bm1;  // bitmap word t of tokens g, g+8
};

// Coherent cached loads (ld.global.ca, not the read-only .nc path): in a fused decode step
// the last block of a unit was written earlier in the same launch, and the acquire in
// wait_ready must order these loads after it.
template <int NCH>
__device__ __forceinline__ void load_raw(RawRegs<NCH>& rr, const uint16_t* __restrict__ vals,
                                         const uint64_t* __restrict__ bms, int tok0, int nvalid, int lane) {
  using Gm = PairGeom<NCH>;
  const int tau = lane >> 1, h = lane & 1, g = lane >> 2, t = lane & 3;
  const int m0 = h ? Gm::kp / 2 + 2 : 0;
  // words wb .. wb + nw - 1 of token tok0 + tau, wb = m0/2 - 1 (h = 0: word -1 is zero)
  const bool ok = tau < nvalid;
  auto ld = [](const uint32_t* a) { return __ldca(a); };
  if constexpr (NCH >= 8) {
  // k_pad >= 64: both halves load nw words from an 8-byte aligned start (word 0 / word kp/4)
  // with 64-bit loads, then the lower half shifts by one word (its W[0] is the zero word -1).
  // Half the load instructions and L1 sector lookups of the scalar path (the L1 data pipe is
  // the bound at 50% density); at k_pad 40 the extra selects cost more than they save.
  const uint2* vsrc = reinterpret_cast<const uint2*>(vals + (size_t)(tok0 + tau) * Gm::kp + (h ? Gm::kp / 2 : 0));
  uint32_t T[Gm::nw + 1];
#pragma unroll
  for (int i = 0; i < (Gm::nw + 1) / 2; ++i) {
    const uint2 x = ok ? __ldca(vsrc + i) : make_uint2(0u, 0u);
    T[2 * i] = x.x;
    if (2 * i + 1 < Gm::nw + 1) T[2 * i + 1] = x.y;
  }
  rr.W[0] = h ? T[0] : 0u;
#pragma unroll
  for (int i = 1; i < Gm::nw; ++i) rr.W[i] = h ? T[i] : T[i - 1];
  } else {
  const uint32_t* src = reinterpret_cast<const uint32_t*>(vals + (size_t)(tok0 + tau) * Gm::kp) + (m0 / 2 - 1);
  rr.W[0] = (h && ok) ? ld(src) : 0u;
  // the upper half's last two words lie past the token (they only feed pair entries beyond
  // k_pad, which no gather reads); the values buffers carry a 16-byte tail guard
  // (mstf_cache_buffer_bytes) so the last record's overrun stays inside the allocation
#pragma unroll
  for (int i = 1; i < Gm::nw; ++i) rr.W[i] = ok ? ld(src + i) : 0u;
  }
  const uint32_t* bw = reinterpret_cast<const uint32_t*>(bms);
  rr.bm0 = g < nvalid ? ld(bw + (size_t)(tok0 + g) * 4 + t) : 0u;
  rr.bm1 = g + 8 < nvalid ? ld(bw + (size_t)(tok0 + g + 8) * 4 + t) : 0u;
}

// Absolute shared address of this lane's first pair-array entry (row m0 of its token's column):
// a function of the lane only, computed once per warp (outside the block loop). The V region
// base is picked with selects, not a switch (a runtime switch on a lane-dependent index makes
// the warp diverge).
template <int NCH, bool IS_V>
__device__ __forceinline__ uint32_t pair_dst(const uint8_t* smem, uint32_t ybase, int lane) {
  using Gm = PairGeom<NCH>;
  const int tau = lane >> 1, h = lane & 1;
  const int m0 = h ? Gm::kp / 2 + 2 : 0;
  uint32_t dst;
  if (IS_V) {
    const int r = (tau & 1) + 2 * (tau >> 3);
    using VL = VLayout<NCH>;
    const int reg = r == 0 ? VL::v0 : r == 1 ? VL::v1 : r == 2 ? VL::v2 : VL::v3;
    dst = ybase + 4u * (uint32_t)(reg + ((tau >> 1) & 3) + 4 * m0);
  } else {
    dst = ybase + 4u * (uint32_t)((tau >> 3 ? KLayout<NCH>::k1 : KLayout<NCH>::k0) + (tau & 7) + 8 * m0);
  }
  return dst + smem_u32(smem);
}

template <int NCH, bool IS_V>
__device__ __forceinline__ void store_pairs(uint32_t adst_in, const RawRegs<NCH>& rr) {
  using Gm = PairGeom<NCH>;
  constexpr uint32_t step = IS_V ? 16 : 32;
  const uint32_t adst = opaque(adst_in);
#pragma unroll
  for (int e = 0; e < Gm::E; ++e) {
    const uint32_t y = (e & 1) ? rr.W[(e + 1) >> 1] : prmt(rr.W[e >> 1], rr.W[(e >> 1) + 1], 0x5432);
    sts_abs(adst + step * e, y);
  }
}

// Work schedule (stream-K over warp pairs). A unit's work items are its compressed 16-token
// blocks (ceil(n_comp/16)) followed by its window row blocks (ceil(W/16)); the units' item
// lists are concatenated (N items). A worker is one K/V warp pair (K-warp w, V-warp w+4) and
// NP = 4 * gridDim.x workers run independently (no CTA-wide sync after the prologue):
//   static part: worker P takes items [B(P), B(P+1)), B(P) = floor(P*S/NP), which may cross
//     unit boundaries; its segment (P, u) writes partial slot P + u.
//   dynamic tail: items [S, N) in chunks of sk_c items; a worker that runs out of work
//     grabs the next chunk from an atomic counter (equal-work workers run at data-dependent
//     speeds, measured with tools/trace_ctas.py, so a purely static split ends with its
//     slowest worker); segment (k, u) of chunk k writes slot NP + U + k + u.
// Both slot maps are injective (along a monotone path of (P|k, u) pairs the sum strictly
// increases) and their ranges are disjoint. Unit u's partial slots are those of the workers /
// chunks overlapping it, a pure function of u (unit_parts); mstf_sk_combine_kernel merges them
// (a9) in the next launch (programmatic dependent launch hides its start-up).
// Segments never drain the K -> V pipeline: the K-warp publishes each segment's descriptor
// {unit, lo, hi, slot} into a 2-deep mbarrier-guarded ring and streams on into the next
// segment; the V-warp consumes descriptors in order. Each warp writes its half of the
// partial (K: m, l per head; V: o per head) when it leaves a segment.

// Dev-only CTA timeline (MSTF_TRACE=1): per CTA {start ns, -, smid, -, K-warp end ns [4],
// V-warp end ns [4], segments per worker [4], ...}.
constexpr int kTraceMax = 4096;
constexpr int kTraceW = 24;
__device__ unsigned long long g_trace[kTraceW * kTraceMax];
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// First item of unit u (u = U gives N). Ragged caches read the prefix array the CTA built
// in shared memory; recomputed from the params where needed (no live registers).
__device__ __forceinline__ int unit_start(const AttnParams& p, const uint8_t* smem, int u) {
  return p.sk_nb ? u * p.sk_nb : reinterpret_cast<const int*>(smem + p.off_pref)[u];
}

// Cost model of the stream-K partition: a unit's cost list is [sk_cs start units (no item:
// q reload and pipeline restart)][one unit per compressed block][sk_cw units per window
// block (dense rows, read without software pipelining)]. Workers split the concatenated
// cost lists evenly; an item belongs to the worker whose range holds its first cost unit.
__device__ __forceinline__ int unit_cost(const AttnParams& p, int n_comp, int nwb) {
  return p.sk_cs + (n_comp + 15) / 16 + nwb * p.sk_cw;
}
// Index of the first item whose first cost unit is >= x (x unit-relative).
__device__ __forceinline__ int item_of_cost(const AttnParams& p, int x, int nbc, int nwb) {
  const int y = x - p.sk_cs;
  if (y <= 0) return 0;
  if (y <= nbc) return y;
  return min(nbc + (y - nbc + p.sk_cw - 1) / p.sk_cw, nbc + nwb);
}

// Unit counters as the attention sees them: after the append (host mirror) in a fused step,
// else the device counters.
__device__ __forceinline__ int ncomp_of(const AttnParams& p, int u) { return p.fuse ? p.unc : p.c.n_comp[u]; }
__device__ __forceinline__ int nwin_of(const AttnParams& p, int u) { return p.fuse ? p.unw : p.c.n_win[u]; }

// Fused step: wait until the warp that appended this unit's tensor published it.
// The appending warp runs at the start of a lower-indexed CTA, so the wait is short; a bounded
// spin (~1 s) turns a broken invariant into a launch error (trap) instead of a hung GPU.
__device__ __forceinline__ void wait_ready(const int* flag, int epoch, int lane) {
  if (lane == 0) {
    int v;
    for (uint32_t it = 0;; ++it) {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
      if (v == epoch) break;
      if (it > (1u << 22)) __trap();
      __nanosleep(64);
    }
  }
  __syncwarp();
}
__device__ __forceinline__ void publish_ready(int* flag, int epoch) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
}

// Fire-and-forget bulk prefetch into L2 (the window rows of a unit, read after its
// compressed blocks without software pipelining).
__device__ __forceinline__ void l2_prefetch(const void* ptr, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes) : "memory");
}

// Unit containing item `it`.
__device__ __forceinline__ int unit_of_item(const AttnParams& p, const uint8_t* smem, int it) {
  if (p.sk_nb) return it / p.sk_nb;
  int lo = 0, hi = p.c.U;  // largest u with start(u) <= it
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (unit_start(p, smem, mid) <= it) lo = mid; else hi = mid;
  }
  return lo;
}

// Static partition: worker P owns cost units [B(P), B(P+1)), B(P) = floor(P * S / NP), so
// every worker gets floor or ceil of S / NP; the owner of unit x is floor(((x+1)*NP - 1) / S).
__device__ __forceinline__ int worker_begin(const AttnParams& p, int P) {
  return (int)((long long)P * p.sk_static / p.sk_np);
}
__device__ __forceinline__ int worker_of(const AttnParams& p, int x) {
  return (int)(((long long)(x + 1) * p.sk_np - 1) / p.sk_static);
}
// Partial slots of unit u (first cost unit us, end ue): static workers, then tail chunks,
// overlapping it.
__device__ __forceinline__ PartRanges unit_parts(const AttnParams& p, int u, int us, int ue) {
  const int NP = p.sk_np;
  const int s_end = p.sk_static;
  PartRanges r{0, 0, 0, 0};
  if (us < s_end) {
    const int cf = worker_of(p, us), cl = worker_of(p, min(ue, s_end) - 1);
    r.b1 = cf + u;
    r.n1 = cl - cf + 1;
  }
  if (ue > s_end) {
    const int kf = (max(us, s_end) - s_end) / p.sk_c, kl = (ue - 1 - s_end) / p.sk_c;
    r.b2 = NP + p.c.U + kf + u;
    r.n2 = kl - kf + 1;
  }
  return r;
}

template <int NK, int NV>
__global__ void __launch_bounds__(256, 2) mstf_attn_reg_kernel(const AttnParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* hfull = reinterpret_cast<uint64_t*>(smem);  // [pair][2] K -> V block handoff
  uint64_t* hempty = hfull + 8;
  uint64_t* dfull = hfull + 16;                         // [pair][2] segment descriptors
  uint64_t* dempty = hfull + 24;
  uint4* handoff = reinterpret_cast<uint4*>(smem + kBarBytesReg);
  __shared__ int4 s_desc[4][2];                         // {unit, lo, hi, slot}; unit < 0: end

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const CacheView& c = p.c;
  const int nwb = c.W > 0 ? (c.W + 15) / 16 : 0;  // window row blocks per unit
  const int cta = blockIdx.x;
  const bool tracing = p.trace && cta < kTraceMax;
  if (tracing && threadIdx.x == 0) {
    g_trace[kTraceW * cta] = global_ns();
    g_trace[kTraceW * cta + 2] = smid();
    for (int i = 3; i < kTraceW; ++i) g_trace[kTraceW * cta + i] = 0;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 32; ++i) mbar_init(&hfull[i], 1);
    fence_mbar_init();
  }
  pdl_launch_dependents();
  pdl_wait();  // cache, counters and q may be written by the previous kernel in the stream
  if (p.sk_nb == 0 && warp == 0) {
    // ragged cache: warp 0 scans the per-unit item counts into smem (CTA 0 also publishes
    // them for the combine kernel)
    int* pref = reinterpret_cast<int*>(smem + p.off_pref);
    int carry = 0;
    for (int u0 = 0; u0 < c.U; u0 += 32) {
      const int uu = u0 + lane;
      const int items = uu < c.U ? unit_cost(p, c.n_comp[uu], nwb) : 0;
      int incl = items;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (uu < c.U) {
        pref[uu] = carry + incl - items;
        if (cta == 0) p.sk_pref[uu] = carry + incl - items;
      }
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      pref[c.U] = carry;
      if (cta == 0) p.sk_pref[c.U] = carry;
    }
  }
  __syncthreads();  // barriers and prefix visible; the only CTA-wide barrier

  const bool is_k = warp < 4;
  const int w = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  const uint32_t ybase = p.off_pairs + (is_k ? (uint32_t)w * p.reg_k : 4 * p.reg_k + (uint32_t)w * p.reg_v);
  const int NP = p.sk_np;
  int blk = 0;   // block handoff sequence number (K-warp w and V-warp w+4 walk the same blocks)
  int nseg = 0;  // segment descriptor sequence number

  if (p.fuse) {
    // fused decode step, a4: worker P appends the new K (K-warp) / V (V-warp) token of units
    // P, P + NP, ... and publishes it; readers wait on the flag (wait_ready) before the blocks
    // the append touched (the evicted token's record, the window ring)
    for (int a = (int)blockIdx.x * 4 + w; a < c.U; a += NP) {
      append_unit_warp(c, is_k ? 0 : 1, a, (is_k ? p.k_new : p.v_new) + (size_t)a * kD, p.nc_old, p.nw_old, lane);
      __syncwarp();
      __threadfence();
      if (lane == 0) {
        if (is_k) {
          if (p.evict) c.n_comp[a] = p.unc; else c.n_win[a] = p.unw;
        }
        publish_ready(p.ready + (is_k ? 0 : c.U) + a, p.epoch);
      }
    }
  }

  if (is_k) {
    // ================= K-warp: schedule, scores + online softmax, P^T -> V-warp
    // Bookkeeping in shared memory, written by lane 0 (keeps it out of registers): [0] unit,
    // [1] next item, [2] range end, [3] lo, [4] hi (unit-relative), [5] slot base,
    // [6] prefetched tail chunk, [7] more work, [8] unit end (absolute).
    __shared__ int s_seg[4][10];
    volatile int* sg = s_seg[w];
    auto set_bounds = [&]() {  // lane 0: cost range of the segment -> item range [lo, hi)
      const int u0 = sg[0];
      const int us = unit_start(p, smem, u0), ue = unit_start(p, smem, u0 + 1);
      const int nbc0 = (ncomp_of(p, u0) + 15) / 16;
      sg[3] = item_of_cost(p, sg[1] - us, nbc0, nwb);
      sg[4] = item_of_cost(p, min((int)sg[2], ue) - us, nbc0, nwb);
      sg[8] = ue;
    };
    auto publish = [&](int4 d) {  // lane 0: descriptor for the V-warp
      const int ds = nseg & 1;
      if (nseg >= 2) mbar_wait(&dempty[2 * w + ds], ((nseg >> 1) - 1) & 1);
      s_desc[w][ds] = d;
      mbar_arrive(&dfull[2 * w + ds]);
    };
    if (lane == 0) {
      const int P = (int)blockIdx.x * 4 + w;
      const int it0 = worker_begin(p, P), it1 = worker_begin(p, P + 1);
      sg[7] = it0 < it1;
      if (sg[7]) {
        sg[1] = it0;
        sg[2] = it1;
        sg[0] = unit_of_item(p, smem, it0);
        sg[5] = P;
        set_bounds();
      }
      // first tail grab now: its latency hides behind the static range
      sg[6] = p.sk_nchunks > 0 ? atomicAdd(p.sk_ctr, 1) : 0;
    }
    __syncwarp();
    KState st;
    int qu = -1;  // unit whose q is in st.qf
    for (;;) {
      if (lane == 0) publish(sg[7] ? make_int4(sg[0], sg[3], sg[4], sg[5] + sg[0]) : make_int4(-1, 0, 0, 0));
      ++nseg;
      __syncwarp();
      if (!sg[7]) break;
      const int u = sg[0];
      const int n = ncomp_of(p, u);
      const int nbc = (n + 15) / 16;
      const int bbeg = min((int)sg[3], nbc), bend = min((int)sg[4], nbc);
      if (lane == 0 && (int)sg[4] > nbc) l2_prefetch(c.win[0] + (size_t)u * c.W * kD, (uint32_t)c.W * kD * 2);
      st.m0 = st.m1 = -INFINITY;
      st.l0 = st.l1 = 0.f;
      if (u != qu) {
        qu = u;
        if (g < p.G) {
          const uint4* qp = reinterpret_cast<const uint4*>(p.q + ((size_t)u * p.G + g) * kD + 32 * t);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint4 x = qp[i];
            st.qf[4 * i] = x.x; st.qf[4 * i + 1] = x.y; st.qf[4 * i + 2] = x.z; st.qf[4 * i + 3] = x.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) st.qf[i] = 0;
        }
      }
      auto handoff_put = [&](const uint4 hh) {
        const int hs = blk & 1;
        if (blk >= 2) mbar_wait(&hempty[2 * w + hs], ((blk >> 1) - 1) & 1);
        handoff[(w * 2 + hs) * 32 + lane] = hh;
        __syncwarp();
        if (lane == 0) mbar_arrive(&hfull[2 * w + hs]);
        ++blk;
      };
      {
        // unit base pointers are re-derived per load (sg[0], params) to save registers
        const size_t ub = (size_t)u * c.cap;
        const uint16_t* const vbase = c.val[0] + ub * c.kpad[0];
        const uint64_t* const bbase = c.bm[0] + ub * kTiles;
        const int wait_blk = (p.fuse && p.evict) ? nbc - 1 : -1;
        auto load = [&](RawRegs<NK>& rr, int bb) {
          // the last block holds the record the fused append wrote: wait for its flag
          if (bb == wait_blk) wait_ready(p.ready + u, p.epoch, lane);
          load_raw<NK>(rr, vbase, bbase, bb * 16, min(16, n - bb * 16), lane);
        };
        // One loop body (not a two-way unrolled ping-pong): the kernel's code footprint is what
        // the instruction cache sees with K- and V-warps resident together. One raw buffer:
        // once a block's words are in the pair array its registers are dead, so the next
        // block's loads go into them right away and overlap the gathers, MMAs and softmax.
        RawRegs<NK> rr;
        const uint32_t pdst = pair_dst<NK, false>(smem, ybase, lane);
        int b = bbeg;
        if (b < bend) load(rr, b);
#pragma unroll 1
        for (; b < bend; ++b) {
          const int nvalid = min(16, n - b * 16);
          __syncwarp();
          store_pairs<NK, false>(pdst, rr);
          const uint32_t bm0 = rr.bm0, bm1 = rr.bm1;
          if (b + 1 < bend) load(rr, b + 1);
          const uint32_t pk = __popc(bm0) | (__popc(bm1) << 16);
          uint32_t ik = pk;
#pragma unroll
          for (int o = 1; o < 4; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, ik, o, 4);
            if (t >= o) ik += y;
          }
          const uint32_t ek = ik - pk;
          __syncwarp();
          uint32_t kr[2][16];
          gather16_s<32>(smem, bm0, ybase + 4u * (uint32_t)(KLayout<NK>::k0 + g) + 32u * (ek & 0xFFFF), kr[0]);
          gather16_s<32>(smem, bm1, ybase + 4u * (uint32_t)(KLayout<NK>::k1 + g) + 32u * (ek >> 16), kr[1]);
          handoff_put(k_block(kr, g < nvalid, g + 8 < nvalid, st, p.scale_log2));
        }
      }
      const int nw = nwin_of(p, u), first = c.W > 0 ? n % c.W : 0;
      if (p.fuse && max((int)sg[3], nbc) < (int)sg[4]) wait_ready(p.ready + u, p.epoch, lane);
      for (int x = max((int)sg[3], nbc), hi = sg[4]; x < hi; ++x) {
        DenseBlock db;
        db.k = c.win[0] + (size_t)u * c.W * kD;
        db.v = c.win[1] + (size_t)u * c.W * kD;
        db.ring = true; db.row0 = (x - nbc) * 16; db.nvalid = 0; db.W = c.W; db.first = first; db.nwin = nw;
        bool any = false;
#pragma unroll
        for (int rr = 0; rr < 16; ++rr) any |= db.valid(rr);
        if (!any) continue;
        uint32_t kr[2][16];
#pragma unroll
        for (int xx = 0; xx < 2; ++xx) {
          const int tok = g + 8 * xx;
          if (db.valid(tok)) {
            const uint4* pp = reinterpret_cast<const uint4*>(db.k + (size_t)(db.row0 + tok) * kD + 32 * t);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint4 a4 = __ldcg(pp + j);
              kr[xx][4 * j] = a4.x; kr[xx][4 * j + 1] = a4.y; kr[xx][4 * j + 2] = a4.z; kr[xx][4 * j + 3] = a4.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) kr[xx][j] = 0;
          }
        }
        handoff_put(k_block(kr, db.valid(g), db.valid(g + 8), st, p.scale_log2));
      }
      float l0 = st.l0, l1 = st.l1;
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
      }
      float* ml = p.ws_ml + (size_t)(sg[5] + u) * p.G * 2;
      if (g == 0) {
        if (2 * t < p.G) { ml[4 * t] = st.m0; ml[4 * t + 1] = l0; }
        if (2 * t + 1 < p.G) { ml[4 * t + 2] = st.m1; ml[4 * t + 3] = l1; }
      }
      __syncwarp();
      if (lane == 0) {
        if (tracing) g_trace[kTraceW * cta + 12 + w] += 1;  // segments of worker w
        // advance: rest of the range in the next unit, else the next tail chunk, else done
        if (sg[2] > sg[8]) {
          sg[1] = sg[8];
          sg[0] = sg[0] + 1;
          set_bounds();
        } else if (p.sk_nchunks > 0 && sg[6] < p.sk_nchunks) {
          const int k = sg[6];
          const int it0 = p.sk_static + k * p.sk_c;
          sg[1] = it0;
          sg[2] = min(it0 + p.sk_c, p.sk_total);
          sg[0] = unit_of_item(p, smem, it0);
          sg[5] = NP + c.U + k;
          set_bounds();
          sg[6] = atomicAdd(p.sk_ctr, 1);  // prefetch the following chunk
        } else {
          sg[7] = 0;
          if (p.sk_nchunks > 0 && atomicAdd(p.sk_ctr + 1, 1) == NP - 1) {
            // last worker to run out: every grab has happened; reset for the next call
            p.sk_ctr[0] = 0;
            p.sk_ctr[1] = 0;
          }
        }
      }
      __syncwarp();
    }
    if (tracing && lane == 0) g_trace[kTraceW * cta + 4 + w] = global_ns();  // K-warp w done
  } else {
    // ================= V-warp: P.V over the segments the K-warp publishes
    for (;;) {
      const int ds = nseg & 1;
      mbar_wait(&dfull[2 * w + ds], (nseg >> 1) & 1);
      const int4 d = s_desc[w][ds];
      __syncwarp();
      if (lane == 0) mbar_arrive(&dempty[2 * w + ds]);
      ++nseg;
      const int u = d.x;
      if (u < 0) {
        if (tracing && lane == 0) g_trace[kTraceW * cta + 8 + w] = global_ns();  // V-warp w done
        break;
      }
      const int n = ncomp_of(p, u);
      const int nbc = (n + 15) / 16;
      const int bbeg = min(d.y, nbc), bend = min(d.z, nbc);
      if (lane == 0 && d.z > nbc) l2_prefetch(c.win[1] + (size_t)u * c.W * kD, (uint32_t)c.W * kD * 2);
      float acc[2][4][4];
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[e][i][0] = acc[e][i][1] = acc[e][i][2] = acc[e][i][3] = 0.f;
      auto handoff_get = [&]() -> uint4 {
        const int hs = blk & 1;
        mbar_wait(&hfull[2 * w + hs], (blk >> 1) & 1);
        const uint4 hh = handoff[(w * 2 + hs) * 32 + lane];
        __syncwarp();
        if (lane == 0) mbar_arrive(&hempty[2 * w + hs]);
        ++blk;
        return hh;
      };
      {
        // unit base pointers are re-derived per load (saves registers in the hot loop)
        const size_t ub = (size_t)u * c.cap;
        const uint16_t* const vbase = c.val[1] + ub * c.kpad[1];
        const uint64_t* const bbase = c.bm[1] + ub * kTiles;
        const int wait_blk = (p.fuse && p.evict) ? nbc - 1 : -1;
        auto load = [&](RawRegs<NV>& rr, int bb) {
          // the last block holds the record the fused append wrote: wait for its flag
          if (bb == wait_blk) wait_ready(p.ready + c.U + u, p.epoch, lane);
          load_raw<NV>(rr, vbase, bbase, bb * 16, min(16, n - bb * 16), lane);
        };
        // one raw buffer: refilled with the next block as soon as this block's pair array and
        // bitmap words are extracted (see the K-warp loop)
        RawRegs<NV> rr;
        const uint32_t pdst = pair_dst<NV, true>(smem, ybase, lane);
        int b = bbeg;
        if (b < bend) load(rr, b);
#pragma unroll 1
        for (; b < bend; ++b) {
          __syncwarp();
          store_pairs<NV, true>(pdst, rr);
          const uint32_t pv = __popc(rr.bm0) | (__popc(rr.bm1) << 16);
          uint32_t iv = pv;
#pragma unroll
          for (int o = 1; o < 4; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, iv, o, 4);
            if (t >= o) iv += y;
          }
          const uint32_t ev = iv - pv;
          const int sa = 8 * t + (g >> 1), sb = sa + 4;
          const uint32_t w2t = __shfl_sync(0xffffffffu, rr.bm0, sa), w2t8 = __shfl_sync(0xffffffffu, rr.bm1, sa);
          const uint32_t w2t1 = __shfl_sync(0xffffffffu, rr.bm0, sb), w2t9 = __shfl_sync(0xffffffffu, rr.bm1, sb);
          const uint32_t pa = __shfl_sync(0xffffffffu, ev, sa), pb = __shfl_sync(0xffffffffu, ev, sb);
          if (b + 1 < bend) load(rr, b + 1);
          __syncwarp();
          const uint32_t ws[4] = {w2t, w2t1, w2t8, w2t9};
          const uint32_t ps[4] = {pa & 0xFFFF, pb & 0xFFFF, pa >> 16, pb >> 16};
          uint32_t vr[4][8];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const uint32_t base = smem_u32(smem) + ybase + 4u * (uint32_t)(VLayout<NV>::region(x) + t) + 16u * ps[x];
            gather8_il<16>(ws[x], opaque(base), g & 1, vr[x]);
          }
          v_block(vr, handoff_get(), acc);
        }
      }
      const int nw = nwin_of(p, u), first = c.W > 0 ? n % c.W : 0;
      if (p.fuse && max(d.y, nbc) < d.z) wait_ready(p.ready + c.U + u, p.epoch, lane);
      for (int x = max(d.y, nbc); x < d.z; ++x) {
        DenseBlock db;
        db.k = c.win[0] + (size_t)u * c.W * kD;
        db.v = c.win[1] + (size_t)u * c.W * kD;
        db.ring = true; db.row0 = (x - nbc) * 16; db.nvalid = 0; db.W = c.W; db.first = first; db.nwin = nw;
        bool any = false;
#pragma unroll
        for (int rr = 0; rr < 16; ++rr) any |= db.valid(rr);
        if (!any) continue;
        uint32_t vr[4][8];
        const int tk[4] = {2 * t, 2 * t + 1, 2 * t + 8, 2 * t + 9};
#pragma unroll
        for (int x4 = 0; x4 < 4; ++x4) {
          if (db.valid(tk[x4])) {  // interleaved channel order (see gather8_il)
            const uint32_t* pp = reinterpret_cast<const uint32_t*>(db.v + (size_t)(db.row0 + tk[x4]) * kD) +
                                 16 * (g >> 1) + (g & 1);
#pragma unroll
            for (int j = 0; j < 8; ++j) vr[x4][j] = __ldcg(pp + 2 * j);
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) vr[x4][j] = 0;
          }
        }
        v_block(vr, handoff_get(), acc);
      }
      float* o = p.ws_o + (size_t)d.w * p.G * kD;
      // m-tile i, row g <-> channels 32(g>>1) + 4i + 2(g&1) (+1: odd accumulator); row g+8: +16
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int h = 2 * t + hh;
        if (h < p.G) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int ch = 32 * (g >> 1) + 4 * i + 2 * (g & 1);
            *reinterpret_cast<float2*>(o + h * kD + ch) = make_float2(acc[0][i][hh], acc[1][i][hh]);
            *reinterpret_cast<float2*>(o + h * kD + ch + 16) = make_float2(acc[0][i][2 + hh], acc[1][i][2 + hh]);
          }
        }
      }
    }
  }
}

// a9 for the stream-K schedule: one CTA (G warps) per unit merges the unit's partial slots
// (unit_parts). Phase 1: lanes load (m, l) of different slots in parallel and reduce the max
// with shuffles; phase 2: a branch-free loop accumulates w_i * o_i (weights broadcast from
// the lane that holds them), so the slot loads of successive iterations overlap.
// S = blockDim.x / (32 G) sub-warps per head split the unit's slots (S > 1 when a unit has many
// slots, i.e. few units: at batch 1 a unit holds ~70 partials); sub-warp results meet in shared
// memory and sub-warp 0 finishes.
constexpr int kCombineMaxSub = 4;
constexpr int kCombineMaxThreads = 512;  // keeps 128 registers per thread (the 16-slot batch)
template <bool SUB>  // false: one warp per head (S = 1, the many-unit case), exactly the plain loop
__global__ void __launch_bounds__(SUB ? kCombineMaxThreads : kMaxGroup * 32) mstf_sk_combine_kernel(const AttnParams p) {
  pdl_launch_dependents();
  pdl_wait();  // partials come from the attention kernel just before
  extern __shared__ __align__(16) float s_comb[];  // (S - 1) x G x kD accumulators, then (S - 1) x G (m, l)
  const int G = p.G;
  const int u = blockIdx.x, wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = SUB ? wi % G : wi, sub = SUB ? wi / G : 0, S = SUB ? blockDim.x / (32 * G) : 1;
  if (!SUB && h >= G) return;
  const int us = p.sk_nb ? u * p.sk_nb : p.sk_pref[u];
  const int ue = p.sk_nb ? (u + 1) * p.sk_nb : p.sk_pref[u + 1];
  const PartRanges r = unit_parts(p, u, us, ue);
  const int np = r.n1 + r.n2;
  const int i_lo = np * sub / S, i_hi = np * (sub + 1) / S;
  auto slot = [&](int i) -> size_t { return i < r.n1 ? (size_t)(r.b1 + i) : (size_t)(r.b2 + i - r.n1); };
  float m_max = -INFINITY, l_sum = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  constexpr int kB = 16;  // slots per batch: all their loads are issued before any math
  for (int i0 = i_lo; i0 < i_hi; i0 += kB) {
    const int cnt = min(kB, i_hi - i0);
    float2 ml = make_float2(-INFINITY, 0.f);
    if (lane < cnt) ml = *reinterpret_cast<const float2*>(p.ws_ml + (slot(i0 + lane) * G + h) * 2);
    float4 v[kB];
#pragma unroll
    for (int i = 0; i < kB; ++i)
      v[i] = i < cnt ? *(reinterpret_cast<const float4*>(p.ws_o + (slot(i0 + i) * G + h) * kD) + lane)
                     : make_float4(0.f, 0.f, 0.f, 0.f);
    float mb = ml.x;
#pragma unroll
    for (int o = 16; o; o >>= 1) mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, o));
    const float mn = fmaxf(m_max, mb);
    if (mn == -INFINITY) continue;  // warp-uniform: no tokens in this batch nor before
    const float a = exp2f(m_max - mn);
    const float wgt = ml.x == -INFINITY ? 0.f : exp2f(ml.x - mn);
    float lb = wgt * ml.y;
#pragma unroll
    for (int o = 16; o; o >>= 1) lb += __shfl_xor_sync(0xffffffffu, lb, o);
    l_sum = l_sum * a + lb;
    acc.x *= a; acc.y *= a; acc.z *= a; acc.w *= a;
    m_max = mn;
#pragma unroll
    for (int i = 0; i < kB; ++i) {
      const float wi2 = __shfl_sync(0xffffffffu, wgt, i);
      acc.x += wi2 * v[i].x; acc.y += wi2 * v[i].y; acc.z += wi2 * v[i].z; acc.w += wi2 * v[i].w;
    }
  }
  if (SUB && S > 1) {
    float* s_acc = s_comb;                                              // [S-1][G][kD]
    float2* s_ml = reinterpret_cast<float2*>(s_comb + (S - 1) * G * kD);  // [S-1][G]
    if (sub > 0) {
      *reinterpret_cast<float4*>(s_acc + ((sub - 1) * G + h) * kD + 4 * lane) = acc;
      if (lane == 0) s_ml[(sub - 1) * G + h] = make_float2(m_max, l_sum);
    }
    __syncthreads();
    if (sub > 0) return;
    for (int j = 0; j < S - 1; ++j) {
      const float2 o = s_ml[j * G + h];
      const float mn = fmaxf(m_max, o.x);
      if (mn == -INFINITY) continue;
      const float a = exp2f(m_max - mn), b2 = exp2f(o.x - mn);
      const float4 x = *reinterpret_cast<const float4*>(s_acc + (j * G + h) * kD + 4 * lane);
      acc.x = acc.x * a + x.x * b2; acc.y = acc.y * a + x.y * b2;
      acc.z = acc.z * a + x.z * b2; acc.w = acc.w * a + x.w * b2;
      l_sum = l_sum * a + o.y * b2;
      m_max = mn;
    }
  }
  const size_t oi = ((size_t)u * G + h) * kD + 4 * lane;
  if (p.part_ml) {  // sequence-split shard: unnormalised partials (log2 domain)
    *reinterpret_cast<float4*>(p.part_o + oi) = acc;
    if (lane == 0) *reinterpret_cast<float2*>(p.part_ml + ((size_t)u * G + h) * 2) = make_float2(m_max, l_sum);
    return;
  }
  const float inv = 1.f / l_sum;
  if (p.out_f16) {
    __half2* po = reinterpret_cast<__half2*>(reinterpret_cast<__half*>(p.out) + oi);
    po[0] = __floats2half2_rn(acc.x * inv, acc.y * inv);
    po[1] = __floats2half2_rn(acc.z * inv, acc.w * inv);
  } else {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + oi) =
        make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  }
}

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
int32_t max_splits_for(int32_t U, int32_t capacity) {
  const int32_t chunks = (capacity + kChunk - 1) / kChunk;
  int32_t s = (8 * 148 + U - 1) / U;  // plan_attention: <= ~4 waves of 2 CTAs per SM (148 SMs)
  if (s > 64) s = 64;
  if (s > chunks) s = chunks;
  return s < 1 ? 1 : s;
}

// Workspace header: [U] unit tickets (kv kernel) + [2] stream-K tail counters (zero between
// calls), the stream-K per-unit prefix [U+1], the fused step's ready flags [2U].
static size_t round256(size_t b) { return (b + 255) / 256 * 256; }
static size_t ticket_bytes(int32_t U) {
  return round256((size_t)(U + 2) * sizeof(int)) + round256((size_t)(U + 1) * sizeof(int)) +
         round256((size_t)2 * U * sizeof(int));
}

size_t attention_ws_bytes(int32_t U, int32_t G, int32_t max_splits) {
  // split grid (TMA kernel): U*S*4 per-warp partials; stream-K (register kernel): one partial
  // per slot, at most NP + U (static) + chunks + U (tail), NP = 4 * grid <= 4 * kMaxSkGrid and
  // chunks <= kSkChunksPerWorker * NP
  size_t parts = (size_t)U * max_splits * kConsumerWarps;
  const size_t np = 4 * (size_t)kMaxSkGrid;
  const size_t sk_parts = 2 * (size_t)U + np * (1 + kSkChunksPerWorker) + 1;
  if (parts < sk_parts) parts = sk_parts;
  return ticket_bytes(U) + parts * G * (kD + 2) * sizeof(float) + 256;
}

// Bytes of one warp's pair-array region: max of the contiguous layout (generic kernels) and
// the interleaved layout (templated kernels), rounded to 128 B (bank offset 0).
static int32_t pair_region_bytes(int32_t kp, bool v) {
  const int32_t contiguous = 16 * (4 * kp + 16);
  const int32_t rows = kp + 4;
  int32_t words;
  if (!v) {
    const int32_t k1 = pad_to_bank(8 * rows, 8);
    words = k1 + 8 * rows;
  } else {
    const int32_t v1 = pad_to_bank(4 * rows, 4);
    const int32_t v2 = pad_to_bank(v1 + 4 * rows, 16);
    const int32_t v3 = pad_to_bank(v2 + 4 * rows, 20);
    words = v3 + 4 * rows;
  }
  const int32_t inter = 4 * words;
  const int32_t b = contiguous > inter ? contiguous : inter;
  return (b + 127) / 128 * 128;
}

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

// Register-staged kernel (stream-K + combine kernel) for equal K/V k_pad of 16, 32, 40 or 64;
// the TMA-staged kernel + separate combine otherwise.
bool uses_reg_kernel(int32_t kpad_k, int32_t kpad_v) {
  const int32_t nk = kpad_k / 8;
  return kpad_k == kpad_v && (nk == 2 || nk == 4 || nk == 5 || nk == 8);
}

AttnPlan plan_attention(int32_t U, int32_t max_comp, int64_t total_items, int32_t uniform_items,
                        int32_t kpad_k, int32_t kpad_v, int32_t sm_count) {
  AttnPlan pl;
  pl.stage_bytes = kChunk * (16 + 2 * kpad_k + 16 + 2 * kpad_v);
  pl.reg_k = pair_region_bytes(kpad_k, false);
  pl.reg_v = pair_region_bytes(kpad_v, true);
  pl.pair_bytes = kConsumerWarps * (pl.reg_k + pl.reg_v);
  // two CTAs per SM when it fits: ~110 KB per CTA for stages + pair arrays
  int ns = (110 * 1024 - pl.pair_bytes - 256 - 4096) / pl.stage_bytes;
  pl.nstage = ns < 2 ? 2 : (ns > 4 ? 4 : ns);
  const int32_t chunks = (max_comp + kChunk - 1) / kChunk;
  // Split count: minimise waves(U*S / (2 CTAs per SM)) x (chunks per CTA + c0), where c0 ~ 2 chunks
  // is the measured per-CTA fixed cost (prologue, first loads, epilogue; tools/split_scan.py).
  const int32_t slots = 2 * sm_count;
  const int32_t cap_s = chunks > 1 ? chunks : 1;
  int32_t best = 1;
  double best_t = 1e30;
  const int32_t max_s = (4 * slots + U - 1) / U;  // at most ~4 waves
  for (int32_t s = 1; s <= cap_s && s <= max_s && s <= 64; ++s) {
    const double waves = std::ceil((double)U * s / slots);
    const double t = waves * ((double)chunks / s + 2.0);
    if (t < best_t - 1e-9) { best_t = t; best = s; }
  }
  pl.splits = best;
  // Stream-K schedule for the register-staged kernel (see the schedule comment above the
  // kernel): one wave of 2 CTAs per SM = 8 warp-pair workers per SM; each worker gets a
  // static (100 - tail)% share of the items, the rest is handed out as dynamic chunks
  // (<= kSkChunksPerWorker per worker). Ragged units need a (U+1)-int prefix array in shared
  // memory, so very large ragged U falls back to the TMA kernel's split grid.
  pl.sk = 0;
  pl.sk_static = pl.sk_nb = pl.sk_grid = pl.sk_c = pl.sk_nchunks = 0;
  pl.sk_total = 0;
  if (uses_reg_kernel(kpad_k, kpad_v) && total_items > 0 && total_items < (1ll << 30) &&
      (uniform_items > 0 || U <= kMaxSkPrefix)) {
    int64_t grid = 2 * (int64_t)sm_count;
    if (const char* e = std::getenv("MSTF_SKGRID")) grid = std::atoi(e);  // dev: occupancy scan
    if (grid > kMaxSkGrid) grid = kMaxSkGrid;
    // >= 14 cost units per CTA (3.5 per worker) to amortise each worker's segment prologue and
    // keep the combine's partials per unit few: at batch 1 (C2 shape, 8 units) this picks 148
    // CTAs instead of 260, 22.6 -> 19.3 us per step (tools/grid_scan.py); from batch 2 up the
    // grid stays at 2 CTAs per SM
    const int64_t min_q = 14;
    if (grid > (total_items + min_q - 1) / min_q) grid = (total_items + min_q - 1) / min_q;
    if (grid < 1) grid = 1;
    const int64_t np = 4 * grid;
    int tail_pct = 0;  // measured: chunk segments cost more than the balance they buy
    if (const char* e = std::getenv("MSTF_SKTAIL")) tail_pct = std::atoi(e);  // tuning override
    int64_t min_chunk = 2;
    if (const char* e = std::getenv("MSTF_SKC")) min_chunk = std::max<int64_t>(1, std::atoi(e));
    const int64_t q = total_items / np;
    int64_t stat = total_items, chunk = 0, nchunks = 0;
    if (tail_pct > 0 && q >= 8) {
      stat = total_items * (100 - tail_pct) / 100;
      const int64_t tail = total_items - stat;
      chunk = std::max(min_chunk, (tail + kSkChunksPerWorker * np - 1) / (kSkChunksPerWorker * np));
      nchunks = (tail + chunk - 1) / chunk;
    }
    pl.sk = 1;
    pl.sk_static = (int32_t)stat;
    pl.sk_grid = (int32_t)grid;
    pl.sk_c = (int32_t)chunk;
    pl.sk_nchunks = (int32_t)nchunks;
    pl.sk_total = (int32_t)total_items;
    pl.sk_nb = uniform_items;
  }
  return pl;
}

cudaError_t launch_sparse_attention(const CacheView& c, const AttnPlan& plan, int32_t G, const uint16_t* q,
                                    float scale, void* out, int32_t out_f16, void* ws, cudaStream_t s,
                                    const FuseArgs* fuse, float* part_ml, float* part_o) {
  if (fuse && !plan.sk) return cudaErrorInvalidValue;  // the fused step needs the register kernel
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
  p.off_pairs = kBarBytesKV + plan.nstage * plan.stage_bytes;
  p.off_handoff = p.off_pairs + plan.pair_bytes;
  p.reg_k = plan.reg_k;
  p.reg_v = plan.reg_v;
  // partials: U*S*4 per-warp (TMA kernel, split grid) or one per slot, NP + 2U + chunks
  // (register kernel, stream-K)
  const size_t parts = plan.sk ? 4 * (size_t)plan.sk_grid + 2 * (size_t)c.U + plan.sk_nchunks
                               : (size_t)c.U * plan.splits * kConsumerWarps;
  p.tickets = reinterpret_cast<int*>(ws);  // [U] ticket counters at a fixed place (zero between calls)
  p.ws_o = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + ticket_bytes(c.U));
  p.ws_ml = p.ws_o + parts * G * kD;
  p.out = out;
  p.out_f16 = out_f16;
  p.part_ml = part_ml;
  p.part_o = part_o;
  p.sk = 0;
  p.sk_static = p.sk_nb = p.sk_c = p.sk_nchunks = p.sk_total = 0;
  p.sk_ctr = p.tickets + c.U;
  p.sk_pref = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(ws) + round256((size_t)(c.U + 2) * sizeof(int)));
  p.ready = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(ws) + round256((size_t)(c.U + 2) * sizeof(int)) +
                                   round256((size_t)(c.U + 1) * sizeof(int)));
  p.fuse = fuse != nullptr;
  p.k_new = fuse ? fuse->k_new : nullptr;
  p.v_new = fuse ? fuse->v_new : nullptr;
  p.nc_old = fuse ? fuse->nc_old : 0;
  p.nw_old = fuse ? fuse->nw_old : 0;
  p.unc = fuse ? fuse->unc : 0;
  p.unw = fuse ? fuse->unw : 0;
  p.evict = fuse ? fuse->evict : 0;
  p.epoch = fuse ? fuse->epoch : 0;

  p.sk_np = 0;
  p.off_pref = 0;
  p.trace = std::getenv("MSTF_TRACE") != nullptr;  // dev timeline (tools/trace_ctas.py)

  const int smem = kBarBytesKV + plan.nstage * plan.stage_bytes + plan.pair_bytes + kHandoffBytes;
  // kernel choice: register-staged interleaved kernel for kpad <= 40 (nk <= 5); TMA-staged kernel
  // with contiguous pair arrays for kpad >= 48 (interleaving aliases banks at ~50% density).
  void (*kern)(AttnParams) = mstf_attn_kv_kernel<0, 0, false>;
  const int nk = c.kpad[0] / 8, nv = c.kpad[1] / 8;
  if (nk == nv) {
    switch (nk) {
      case 5: kern = mstf_attn_kv_kernel<5, 5, true>; break;
      case 8: kern = mstf_attn_kv_kernel<8, 8, false>; break;
      case 16: kern = mstf_attn_kv_kernel<16, 16, false>; break;
      default: break;
    }
  }
  if (plan.sk) {  // register-staged kernel, stream-K schedule
    void (*rk)(AttnParams) = nullptr;
    switch (nk) {
      case 2: rk = mstf_attn_reg_kernel<2, 2>; break;
      case 4: rk = mstf_attn_reg_kernel<4, 4>; break;
      case 8: rk = mstf_attn_reg_kernel<8, 8>; break;
      default: rk = mstf_attn_reg_kernel<5, 5>; break;
    }
    AttnParams pr = p;
    pr.off_pairs = kBarBytesReg + kHandoffBytes;
    int rsmem = pr.off_pairs + plan.pair_bytes;
    pr.sk = 1;
    pr.sk_static = plan.sk_static;
    pr.sk_c = plan.sk_c;
    pr.sk_nchunks = plan.sk_nchunks;
    pr.sk_total = plan.sk_total;
    pr.sk_nb = plan.sk_nb;
    pr.sk_np = 4 * plan.sk_grid;
    sk_cost_params(&pr.sk_cs, &pr.sk_cw);
    pr.off_pref = (uint32_t)rsmem;
    if (plan.sk_nb == 0) rsmem += (c.U + 1) * (int)sizeof(int);
    const dim3 grid(plan.sk_grid, 1);
    cudaError_t e = cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, rsmem);
    if (e != cudaSuccess) return e;
    e = launch_pdl(rk, grid, dim3(256), (size_t)rsmem, s, pr);
    if (e != cudaSuccess) return e;
    // sub-warps per head: ~16 partial slots each (one load batch), at most kCombineMaxSub
    const int64_t slots_per_unit = (4 * (int64_t)plan.sk_grid + c.U - 1) / c.U + 2;
    int sub = (int)((slots_per_unit + 15) / 16);
    if (const char* e = std::getenv("MSTF_COMBSUB")) sub = std::atoi(e);  // dev A/B
    sub = std::max(1, std::min(std::min(sub, kCombineMaxSub), kCombineMaxThreads / (32 * G)));
    const size_t csmem = (size_t)(sub - 1) * G * (kD * sizeof(float) + sizeof(float2));
    if (sub == 1) return launch_pdl(mstf_sk_combine_kernel<false>, dim3(c.U), dim3(32 * G), 0, s, pr);
    return launch_pdl(mstf_sk_combine_kernel<true>, dim3(c.U), dim3(32 * G * sub), csmem, s, pr);
  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  e = launch_pdl(kern, dim3(plan.splits, c.U), dim3(kThreadsKV), (size_t)smem, s, p);
  if (e != cudaSuccess) return e;
  return launch_pdl(mstf_combine_kernel, dim3(c.U), dim3(G * 32), 0, s, (const float*)p.ws_o, (const float*)p.ws_ml,
                    (int)(plan.splits * kConsumerWarps), (int)G, out, (int)out_f16, part_ml, part_o);
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

cudaError_t copy_trace(void* host, int n) {
  if (n > kTraceW * kTraceMax) n = kTraceW * kTraceMax;
  return cudaMemcpyFromSymbol(host, g_trace, n * sizeof(unsigned long long));
}

}  // namespace mstf
