// attn_warp.cu -- decode attention directly over the compressed cache (Algorithm 1,
// P:236-261), one self-contained warp per work item: the round-2 kernel.
//
// Every warp of a persistent grid (one CTA per SM) is an independent stream-K worker over the
// concatenated 16-token blocks of all units; small problems give each warp
// at most one block and merge the warps' partials per CTA in shared memory (cta_merge):
//   * its compressed blocks are streamed from HBM by TMA bulk copies (cp.async.bulk, four per
//     block: K bitmaps, K values, V bitmaps, V values -- each a contiguous run of fixed-stride
//     records, R5-R7) into a private 2-stage shared-memory ring; the warp issues them itself
//     two blocks ahead, so the hot loop has no global-load instruction; the copies' operands
//     are made provably warp-uniform (shuffled from lane 0, issued by an elect.sync lane), so
//     ptxas keeps them in uniform registers (MSTF_UNIFORM);
//   * the token's build lane also stores the pair-entry addresses of bitmap words 1-3 (prefix
//     counts) in its row's pad words, which the consumer lanes load (MSTF_PREFIX);
//   * expansion ("load as compressed, compute as dense"): one lane per token rewrites
//     the packed values as a shifted pair array Y[m] = (h[m-1], h[m]); channel pair (2j, 2j+1)
//     of a bitmap word with exclusive prefix e is then ONE aligned 32-bit load
//     Y[e + popc(word & bits <= 2j)], masked by the two bitmap bits;
//   * a5 (q.K^T) and a8 (P.V) on the tensor cores (mma.sync m16n8k16, fp16 x fp16 -> fp32),
//     both in the same warp (no K -> V hand-off):
//       scores  S^T[tok][col] = K[tok][ch] . q^T[ch][col]: M = 16 tokens, N = 8 head columns
//               (heads col & 3 duplicated for G <= 4, heads col for G = 8), K = 16 channels;
//               the gathered channel pairs are the A operand as they are;
//       values  O'[pair][(h, p)] = V'[pair][(tok, e)] . P'[(tok, e)][(h, p)], M = 16 channel
//               pairs, K = 8 tokens x 2 parities, N = 4 heads x 2 parities, with
//               P'[(tok, e)][(h, p)] = P[h][tok] if e == p else 0: every A register is one
//               token's gathered channel pair, D[pair][(h, p)] = O[h][2 pair + p]; movmatrix
//               turns the P^T tile of the scores into this B operand;
//   * a7 online softmax in the log2 domain (exp2, log2e folded into the scale);
//   * the dense local window (a6) is read with 128-bit loads in the same loop;
//   * each (worker, unit) segment writes one partial (m, l, o) slot; the combine kernel (a9)
//     merges a unit's slots.
//
// Fused decode step (mstf_decode_step, uniform caches): the workers that own a unit's two start
// cost units append its new K and V token (a4) before their attention work and count a ready
// flag up; a worker reading the unit's last record or its window waits for both. The
// appenders' indices are never higher than a reader's, so in-order CTA dispatch cannot
// deadlock. Counters are read from the device and NOT written here (the combine kernel
// writes the post-append counters and clears the flags), so a captured CUDA graph of the
// step replays correctly.
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "compress_dev.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace mstf {

namespace {

#ifndef MSTF_B128
#define MSTF_B128 1  // pair arrays written with 16-byte stores (dev A/B: 0 = 4-byte stores)
#endif
#ifndef MSTF_PREFIX
#define MSTF_PREFIX MSTF_B128  // per-word pair-entry addresses stored by the build lanes (needs MSTF_B128)
#endif
#ifndef MSTF_UNIFORM
#define MSTF_UNIFORM 1  // per-warp scalars made provably warp-uniform (dev A/B: 0)
#endif
#ifndef MSTF_ZBM
#define MSTF_ZBM 1  // bitmap slots past a partial block's end zeroed in the stage (dev A/B: 0 = predicated loads)
#endif
#ifndef MSTF_BOUNDS
#define MSTF_BOUNDS 0
#endif
#ifndef MSTF_PREFIX_PACK
#define MSTF_PREFIX_PACK 0  // 1: the three prefix counts packed in one word (dev A/B; slower, DESIGN 8.1)
#endif
#ifndef MSTF_PREFIX_SEL
#define MSTF_PREFIX_SEL 3  // which token preps load the stored addresses: bit 0 = K, bit 1 = V (dev A/B)
#endif
#if MSTF_PREFIX && !MSTF_B128
#error "MSTF_PREFIX stores the prefix addresses in the pad words of the 16-byte-store row layout"
#endif
constexpr int kWNst = 2;          // TMA ring depth per warp (blocks in flight)
#ifndef MSTF_PREISSUE
#define MSTF_PREISSUE 1
#endif
// stages issued before the first block is consumed (the rest once the first block has landed:
// the first blocks of all workers then share the HBM fill alone; fp16 payload only -- the 4-bit
// payload measured faster with both stages at entry, C4_q4 531.8 vs 541.1 us; dev A/B)
constexpr int kPreIssueF16 = MSTF_PREISSUE < kWNst ? MSTF_PREISSUE : kWNst;
constexpr int kWMaxWarps = 16;    // warps per CTA (one CTA per SM, <= 128 registers per thread)
constexpr int kWHdrInts = 16;
constexpr int kWPartBytes = 4 * 128 * 4 + 4 * 2 * 4;  // a warp's partial in shared memory (G <= 4)
constexpr int kCombBatch = 16;  // combine: partial slots per sub-warp batch (loads in flight)     // workspace header: [0] S (total cost), [1] cost per unit (0: ragged)

struct WParams {
  CacheView c;
  const uint16_t* q;      // [U][G][kD]
  int G;
  float scale_log2;
  float lazy_log2;        // softmax reference-max slack (log2 units; 0: exact running max)
  int np;                 // workers (warps of the grid)
  int wpc;                // warps per CTA
  int cs, cw;             // cost model: per-segment start, per window block
  int uniform;            // every unit has the same counters (closed-form partition)
  int fuse;               // append inside (uniform caches only)
  int kpk, kpv;           // k_pad of K and V
  int rqk, rqv;           // bytes of one token's value record (2 k_pad, or the 4-bit record)
  int stage_bytes, off_kval, off_vbm, off_vval;
  int swk, swv;           // pair-array stride per token (32-bit words)
  int warp_bytes;         // per-warp shared-memory region
  int* hdr;               // workspace header (kWHdrInts ints)
  int* ready;             // [U] fused step: append done (1), cleared by the combine
  int* pref;              // [U+1] ragged cost prefix (written by mstf_cost_prefix_kernel)
  float* ws_o;            // [slots][G][kD] partial o (unnormalised)
  float* ws_ml;           // [slots][G][2] partial (m, l), log2 domain
  int cta_merge;          // small problems (<= 1 cost unit per warp, G <= 4): warp partials stay in
                          // shared memory and the CTA writes one partial per unit (slot CTA + u of ws2)
  float* ws2_o;           // [grid + U + 1][G][kD]
  float* ws2_ml;          // [grid + U + 1][G][2]
  const uint16_t* k_new;  // fused step: [U][kD]
  const uint16_t* v_new;
  // combine
  void* out;
  int out_f16;
  float* part_ml;
  float* part_o;
};

// Development trace (mstf_dev_trace): per worker, global-timer stamps of its phases; null
// (the default) compiles to one predicated-off branch per phase.
// Compiled in only with -DMSTF_TRACE=1 (dev builds: MSTF_NVCC_EXTRA); otherwise the stamps are
// empty functions and mstf_dev_trace returns MSTF_ENOTSUP.
#ifndef MSTF_TRACE
#define MSTF_TRACE 0
#endif
__device__ unsigned long long* g_mstf_trace = nullptr;
constexpr int kTraceSlots = 8;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_at(int worker, int k) {
#if MSTF_TRACE
  unsigned long long* tr = g_mstf_trace;
  if (tr) tr[(size_t)worker * kTraceSlots + k] = gtimer();
#else
  (void)worker;
  (void)k;
#endif
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
// Opaque copy: keeps a precomputed address in a register of its own (the compiler would otherwise
// re-associate base + 4 (e + popc) and spend an add per gather).
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
  asm("mov.b32 %0, %0;" : "+r"(x));
  return x;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void bulk_g2s_u32(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_init_u32(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx_u32(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// Generic-proxy shared reads of a stage must be ordered before the async-proxy (TMA) write
// that refills it.
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// Global data published by another CTA (generic stores + release / acquire) must be visible to
// a TMA read issued after the acquire.
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// elect.sync over the full warp: true on exactly one lane (the lowest, lane 0 here)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void l2_prefetch(const void* ptr, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes) : "memory");
}

// Byte-mask of one channel pair: x has the pair's low bit at the sign bit of byte M, y its high
// bit; prmt's sign-replicate mode turns them into 0xFFFF halves (kept) or 0x0000 (pruned).
template <int M>
__device__ __forceinline__ uint32_t pair_mask(uint32_t x, uint32_t y) {
  constexpr uint32_t lo = 8 | M, hi = 8 | (4 + M);
  return prmt(x, y, lo | (lo << 4) | (hi << 8) | (hi << 12));
}
// One gather: pair entry Y[idx] of a token's pair array (base = its entry e_q, scaled) ANDed with
// the pair's mask. Every lane loads (no predicate): in the consecutive-pair mapping below the
// lanes of one token read a few neighbouring words, so a pruned pair's lane adds no bank slot.
__device__ __forceinline__ uint32_t gather1(uint32_t base, uint32_t cnt, uint32_t mask) {
  return lds32(base + 4u * cnt) & mask;
}

// Per-token, per-word state of the consecutive-pair gathers:
//   x[q] = w_q << sx, y[q] = w_q << (sx - 1): the lane's pair bits at byte sign positions;
//   B[q] = address of pair entry e_q (kept channels of the token before word q).
// The kept count up to and including a pair's low channel is e_q + popc(x[q] << k) for an
// immediate k that drops the bits above it, so Y[e_q + that] is the pair (R8, R6).
struct TokGather {
  uint32_t x[4], y[4], B[4];
#if MSTF_BOUNDS
  uint32_t lo, hi;  // the token's pair entries Y[0..kp]: [lo, hi]
#endif
};
// MSTF_BOUNDS (dev build, -DMSTF_BOUNDS=1): every data-dependent shared-memory address of the
// expansion -- the stored prefix addresses and each gather -- is checked against its token's
// pair-entry range; a violation traps (the GPU parity tests then fail). Used in place of
// compute-sanitizer, which this GPU pool does not allow.
__device__ __forceinline__ void bounds_check(uint32_t a, uint32_t lo, uint32_t hi) {
  if (a < lo || a > hi) __trap();
}
// MSTF_PREFIX: B[1..3] were stored by the token's build lane after its last pair entry (word kp
// of the row, see build_prefix); the lane loads them instead of three popc + add (XU pipe).
template <bool LOAD>
__device__ __forceinline__ void tok_prep(TokGather& tg, const uint4 w, uint32_t base, uint32_t sx, uint32_t kp4) {
  const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#if MSTF_BOUNDS
  tg.lo = base;
  tg.hi = base + kp4;
#endif
#if MSTF_PREFIX
  if (!LOAD) {
    uint32_t b = base;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      tg.x[q] = ww[q] << sx;
      tg.y[q] = ww[q] << (sx - 1);
      tg.B[q] = opaque(b);
      b += 4u * __popc(ww[q]);
    }
    return;
  }
#if MSTF_PREFIX_PACK
  // e_1..e_3 packed in bytes 0..2 of the word after Y[kp]: one 4-byte load (one wavefront for the
  // tokens of a gather instruction) instead of a shared 16-byte load (one per quarter-warp)
  const uint32_t pk = lds32(base + kp4 + 4u);
  uint4 e;
  e.y = base + 4u * (pk & 0xFFu);
  e.z = base + 4u * ((pk >> 8) & 0xFFu);
  e.w = base + 4u * (pk >> 16);
#else
  const uint4 e = lds128(base + kp4);
#endif
#if MSTF_BOUNDS
  bounds_check(e.y, tg.lo, tg.hi);
  bounds_check(e.z, tg.lo, tg.hi);
  bounds_check(e.w, tg.lo, tg.hi);
#endif
  tg.B[0] = base;
  tg.B[1] = e.y;
  tg.B[2] = e.z;
  tg.B[3] = e.w;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    tg.x[q] = ww[q] << sx;
    tg.y[q] = ww[q] << (sx - 1);
  }
#else
  (void)kp4;
  uint32_t b = base;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    tg.x[q] = ww[q] << sx;
    tg.y[q] = ww[q] << (sx - 1);
    tg.B[q] = opaque(b);
    b += 4u * __popc(ww[q]);
  }
#endif
}
// The last pair entry Y[kp] of a token's row and, with MSTF_PREFIX, the addresses of pair entries
// e_1..e_3 (kept channels before bitmap words 1..3) in the three words after it: one 16-byte
// store. bm = the token's bitmap words (zero for a token past the block's end: every address is
// then the row base, inside the region).
__device__ __forceinline__ void build_tail(uint32_t ydst, int nch, uint32_t last, const uint4 bm) {
#if MSTF_PREFIX
  const uint32_t e1 = __popc(bm.x), e2 = e1 + __popc(bm.y), e3 = e2 + __popc(bm.z);
#if MSTF_PREFIX_PACK
  sts128(ydst + 32u * nch, last, e1 | (e2 << 8) | (e3 << 16), 0u, 0u);
#else
  sts128(ydst + 32u * nch, last, ydst + 4u * e1, ydst + 4u * e2, ydst + 4u * e3);
#endif
#else
  (void)bm;
  sts32(ydst + 32u * nch, last);
#endif
}
// K (score A operand): gather slot j = 2s + hh of lane t is pair 8s + 4hh + t, i.e. channels
// 16s + 8hh + 2t, +1 -- the natural m16n8k16 k order. Word q = j >> 2, byte m = j & 3; the
// lane's bit in byte m is bit 8m + 2t, at bit 8m + 7 of x (sx = 7 - 2t).
template <int J>
__device__ __forceinline__ uint32_t gather_k(const TokGather& tg) {
  constexpr int q = J >> 2, m = J & 3;
  const uint32_t cnt = __popc(m == 3 ? tg.x[q] : tg.x[q] << (24 - 8 * m));
#if MSTF_BOUNDS
  bounds_check(tg.B[q] + 4u * cnt, tg.lo, tg.hi);
#endif
  return gather1(tg.B[q], cnt, pair_mask<m>(tg.x[q], tg.y[q]));
}
// V (value A operand): row r (0: g, 1: g + 8) of m-tile mt is pair 16mt + 8r + g, i.e. word mt,
// bit 16r + 2g, at bit 16r + 15 of x (sx = 15 - 2g): byte 1 + 2r.
template <int MT, int R>
__device__ __forceinline__ uint32_t gather_v(const TokGather& tg) {
  const uint32_t cnt = __popc(R ? tg.x[MT] : tg.x[MT] << 16);
#if MSTF_BOUNDS
  bounds_check(tg.B[MT] + 4u * cnt, tg.lo, tg.hi);
#endif
  return gather1(tg.B[MT], cnt, pair_mask<1 + 2 * R>(tg.x[MT], tg.y[MT]));
}

// Shifted pair arrays of the 16 tokens of both tensors in a stage, one token per lane (lanes
// 0-15: K tokens 0-15, lanes 16-31: V tokens 0-15): Y[m] = (h[m-1], h[m]), m = 0..kp
// (h[-1] = h[kp] = 0) at ydst + 4 * (tau * sw + m). Odd entries are the raw words, even ones
// one prmt each; four entries per 16-byte store. With sw = kp + 4 (4 mod 8 words) the 8 lanes of
// every quarter-warp store phase hit 8 distinct 16-byte bank groups. raw = this lane's record.
template <int NCH>
__device__ __forceinline__ void build_token(uint32_t raw, uint32_t ydst, int nch_rt, const uint4 bm) {
  const int nch = NCH ? NCH : nch_rt;
  uint32_t prev = 0;
#pragma unroll
  for (int c = 0; c < (NCH ? NCH : 16); ++c) {
    if (!NCH && c >= nch) break;
    const uint4 a = lds128(raw + 16 * c);
    const uint32_t d = ydst + 32u * c;
#if MSTF_B128
    sts128(d, prmt(prev, a.x, 0x5432), a.x, prmt(a.x, a.y, 0x5432), a.y);
    sts128(d + 16, prmt(a.y, a.z, 0x5432), a.z, prmt(a.z, a.w, 0x5432), a.w);
#else
    sts32(d, prmt(prev, a.x, 0x5432));
    sts32(d + 4, a.x);
    sts32(d + 8, prmt(a.x, a.y, 0x5432));
    sts32(d + 12, a.y);
    sts32(d + 16, prmt(a.y, a.z, 0x5432));
    sts32(d + 20, a.z);
    sts32(d + 24, prmt(a.z, a.w, 0x5432));
    sts32(d + 28, a.w);
#endif
    prev = a.w;
  }
  build_tail(ydst, nch, prmt(prev, 0u, 0x5432), bm);
}

// The same pair arrays from a 4-bit record: [scale f16][zero f16][codes,
// low nibble first]. Each pair of codes becomes fp16 integers through the 1024 + c bit trick
// (exact), then one fp16 FMA per pair reconstructs f16(c * scale + zero) -- the oracle's single
// rounding. nch = kp / 8 code words (8 codes each; codes past k reconstruct to `zero`, which no
// unmasked gather reads).
__device__ __forceinline__ uint32_t hsub2_u(uint32_t a, uint32_t b) {
  __half2 r = __hsub2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t hfma2_u(uint32_t a, uint32_t b, uint32_t c) {
  __half2 r = __hfma2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b), *reinterpret_cast<__half2*>(&c));
  return *reinterpret_cast<uint32_t*>(&r);
}
// One pair of codes (bytes i of the low / high nibble words) -> f16(c * scale + zero) x 2.
__device__ __forceinline__ uint32_t dequant_pair(uint32_t lo, uint32_t hi, int i, uint32_t sc2, uint32_t z2) {
  const uint32_t t = (prmt(lo, hi, (uint32_t)(((4 + i) << 8) | i)) & 0x00FF00FFu) | 0x64006400u;
  return hfma2_u(hsub2_u(t, 0x64006400u), sc2, z2);
}
// Eight values (code word w) -> pair entries Y[8c .. 8c+7] at d; prev = last raw pair word.
__device__ __forceinline__ void q4_word_pairs(uint32_t w, uint32_t sc2, uint32_t z2, uint32_t d, uint32_t& prev) {
  const uint32_t lo = w & 0x0F0F0F0Fu, hi = (w >> 4) & 0x0F0F0F0Fu;
  uint32_t R[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) R[i] = dequant_pair(lo, hi, i, sc2, z2);
#if MSTF_B128
  sts128(d, prmt(prev, R[0], 0x5432), R[0], prmt(R[0], R[1], 0x5432), R[1]);
  sts128(d + 16, prmt(R[1], R[2], 0x5432), R[2], prmt(R[2], R[3], 0x5432), R[3]);
#else
  sts32(d, prmt(prev, R[0], 0x5432));
  sts32(d + 4, R[0]);
  sts32(d + 8, prmt(R[0], R[1], 0x5432));
  sts32(d + 12, R[1]);
  sts32(d + 16, prmt(R[1], R[2], 0x5432));
  sts32(d + 20, R[2]);
  sts32(d + 24, prmt(R[2], R[3], 0x5432));
  sts32(d + 28, R[3]);
#endif
  prev = R[3];
}
template <int NCH>
__device__ __forceinline__ void build_token_q4(uint32_t rec, uint32_t ydst, int nch_rt, const uint4 bm) {
  uint32_t prev = 0;
  if constexpr (NCH > 0) {
    // the whole record in 16-byte loads (records are 16-byte aligned; scalar loads of 32-byte
    // strided records would hit every bank group 4 times)
    constexpr int RQ = (4 * NCH + 4 + 15) / 16 * 16;
    uint32_t wv[RQ / 4];
#pragma unroll
    for (int i = 0; i < RQ / 16; ++i) {
      const uint4 a = lds128(rec + 16 * i);
      wv[4 * i] = a.x; wv[4 * i + 1] = a.y; wv[4 * i + 2] = a.z; wv[4 * i + 3] = a.w;
    }
    const uint32_t sc2 = prmt(wv[0], 0u, 0x1010), z2 = prmt(wv[0], 0u, 0x3232);
#pragma unroll
    for (int c = 0; c < NCH; ++c) q4_word_pairs(wv[1 + c], sc2, z2, ydst + 32u * c, prev);
    build_tail(ydst, NCH, prmt(prev, 0u, 0x5432), bm);
  } else {
    const uint32_t sz = lds32(rec);
    const uint32_t sc2 = prmt(sz, 0u, 0x1010), z2 = prmt(sz, 0u, 0x3232);
    for (int c = 0; c < nch_rt; ++c) q4_word_pairs(lds32(rec + 4 + 4 * c), sc2, z2, ydst + 32u * c, prev);
    build_tail(ydst, nch_rt, prmt(prev, 0u, 0x5432), bm);
  }
}

// ---------------------------------------------------------------- schedule (device side)
// Cost model of the partition (same as the r1 stream-K schedule): a unit's cost list is
// [cs start units][one per compressed 16-token block][cw per window block]; worker P owns
// cost units [P*S/NP, (P+1)*S/NP); an item belongs to the worker holding its first cost unit;
// segment (P, u) writes partial slot P + u (unique: P + u increases along the monotone path).
struct Counters {
  int nc, nw;  // as the attention sees them (after the fused append, if any)
};
__device__ __forceinline__ Counters counters_of(const WParams& p, int u) {
  Counters r;
  r.nc = p.c.n_comp[u];
  r.nw = p.c.n_win[u];
  if (p.fuse) {  // a4: the step's append precedes the attention (R12)
    if (p.c.W == 0 || r.nw == p.c.W) r.nc += 1; else r.nw += 1;
  }
  return r;
}
__device__ __forceinline__ int nwb_of(const WParams& p) { return p.c.W > 0 ? (p.c.W + 15) / 16 : 0; }
__device__ __forceinline__ int cost_of(const WParams& p, int nc) { return p.cs + (nc + 15) / 16 + nwb_of(p) * p.cw; }
__device__ __forceinline__ int unit_start(const WParams& p, int u, int cpu) { return cpu ? u * cpu : p.pref[u]; }
// first item whose first cost unit is >= x (x unit-relative)
__device__ __forceinline__ int item_of_cost(const WParams& p, int x, int nbc) {
  const int y = x - p.cs;
  if (y <= 0) return 0;
  if (y <= nbc) return y;
  return min(nbc + (y - nbc + p.cw - 1) / p.cw, nbc + nwb_of(p));
}
__device__ __forceinline__ int unit_of_cost(const WParams& p, int x, int cpu) {
  if (cpu) return x / cpu;
  int lo = 0, hi = p.c.U;  // largest u with start(u) <= x
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (p.pref[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int worker_begin(const WParams& p, long long S, int P) { return (int)((long long)P * S / p.np); }
// the worker owning cost unit x: the largest P with worker_begin(P) <= x
__device__ __forceinline__ int worker_of(const WParams& p, long long S, int x) {
  return (int)(((long long)(x + 1) * p.np - 1) / S);
}

// Fused step: wait until the unit's append is published (bounded spin: a broken invariant
// becomes a launch error, not a hung GPU).
// ready[u] counts the unit's appended tensors (K and V may be appended by different workers).
__device__ __forceinline__ void wait_ready(const int* flag) {
  int v;
  for (uint32_t it = 0;; ++it) {
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v >= 2) break;
    if (it > (1u << 22)) __trap();
    __nanosleep(64);
  }
}

// ---------------------------------------------------------------- the kernel
// G = 8 holds twice the accumulators and q fragments: at most 8 warps per CTA (<= 255 registers).
template <int NK, int NV, bool G8, bool Q4>
__global__ void __launch_bounds__(G8 ? kWMaxWarps * 16 : kWMaxWarps * 32, 1) mstf_attn_warp_kernel(const WParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int kPreIssue = Q4 ? kWNst : kPreIssueF16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const CacheView& c = p.c;
#if MSTF_UNIFORM
  // The warp index (hence every per-warp scalar) through a shuffle from lane 0: ptxas then knows
  // these values are warp-uniform and keeps the TMA operands in uniform registers (no
  // elect / R2UR broadcast loop around each cp.async.bulk).
  const int P = __shfl_sync(0xffffffffu, (int)blockIdx.x * p.wpc + warp, 0);
#else
  const int P = (int)blockIdx.x * p.wpc + warp;
#endif
  // per-warp region: [stages kWNst x stage_bytes][pairs K 16 x swk words][pairs V][mbarriers]
  const uint32_t wbase = smem_u32(smem) + (uint32_t)((P - (int)blockIdx.x * p.wpc) * p.warp_bytes);
  const uint32_t ypk = wbase + (uint32_t)(kWNst * p.stage_bytes);  // 128-byte aligned
  const uint32_t ypv = ypk + ((64u * (uint32_t)p.swk + 127u) & ~127u) + (MSTF_B128 ? 0u : 4u);
  const uint32_t bar0 = (max(ypv + 64u * (uint32_t)p.swv, ypk + (uint32_t)kWPartBytes) + 7u) & ~7u;
  __shared__ int s_wunit[kWMaxWarps];  // cta_merge: the unit of the warp's partial (-1: none)
  if (lane == 0) s_wunit[warp] = -1;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kWNst; ++s) mbar_init_u32(bar0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  pdl_launch_dependents();
  pdl_wait();  // cache, counters, q and the ragged prefix come from earlier kernels in the stream
  if (lane == 0) trace_at(P, 0);

  // ---- partition (device counters: graph-replay safe)
  int cpu = 0;  // cost per unit (uniform caches)
  long long S;
  const int nc_0 = c.n_comp[0], nw_0 = c.n_win[0];  // unit 0's counters (before a fused append)
  if (p.uniform) {
    cpu = cost_of(p, counters_of(p, 0).nc);
    S = (long long)c.U * cpu;
  } else {
    S = p.pref[c.U];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // for the combine
    p.hdr[0] = (int)S;
    p.hdr[1] = cpu;
  }
  const int x0 = worker_begin(p, S, P), x1 = worker_begin(p, S, P + 1);

  // ---- a4 (fused step): tensor x (0: K, 1: V) of unit u is appended by the owner of the unit's
  // start cost unit min(x, cs - 1) -- with cs >= 2 two workers when the partition splits them
  // (small problems: two otherwise idle warps), one worker doing both otherwise
  // (run after this warp's first TMA issues, so that their latency overlaps the compression)
  auto fused_appends = [&]() {
    if (!p.fuse) return;
    for (int u = max(0, x0 / cpu - 1); u < c.U && u * cpu < x1; ++u) {
      for (int x = 0; x < 2; ++x) {
        const int j = u * cpu + min(x, p.cs - 1);
        if (j < x0 || j >= x1) continue;
        // uniform caches (fuse requires it): unit 0's counters, already read for the partition
        append_unit_warp(c, x, u, (x ? p.v_new : p.k_new) + (size_t)u * kD, nc_0, nw_0, lane);
        __syncwarp();  // orders every lane's record / window stores before lane 0's release
        if (lane == 0) asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p.ready + u), "r"(1) : "memory");
      }
    }
  };
  if (x0 >= x1) {  // no cost unit: no append either
    if (lane == 0) trace_at(P, 1);
    if (!p.cta_merge) return;
  }
  if (x0 < x1) {  // (cta_merge: every warp reaches the CTA merge at the end)

  // ---- block streams: producer (TMA issue, one block ahead) and consumer walk the same
  // sequence of compressed blocks: segment by segment, unit u's blocks [lo, min(hi, nbc)).
  const int u_first = unit_of_cost(p, x0, cpu);
  // producer cursor: unit pu, next block pb, end pbe; pnc = pu's compressed tokens (as the
  // attention sees them), pwait = the block holding the record the fused append writes (-1: none);
  // prec = record index of block pb's first token (u * cap + 16 pb: < 2^32, a cache of 2^32
  // records would not fit in HBM); the four runs' global addresses (K bitmaps, K values, V bitmaps,
  // V values) are formed from it at issue time (one wide multiply-add each)
  int pu = u_first, pb = 0, pbe = 0, pseq = 0, pnc = 0, pwait = -1;
  uint32_t prec = 0;
  bool pdone = false;
  auto seg_bounds = [&](int u, int& lo, int& hi, int& nbc, Counters& cn) {
    cn = counters_of(p, u);
    nbc = (cn.nc + 15) / 16;
    const int us = unit_start(p, u, cpu), ue = unit_start(p, u + 1, cpu);
    lo = item_of_cost(p, max(x0, us) - us, nbc);
    hi = item_of_cost(p, min(x1, ue) - us, nbc);
  };
  auto p_unit = [&]() {  // producer enters unit pu
    int lo, hi, nbc;
    Counters cn;
    seg_bounds(pu, lo, hi, nbc, cn);
    pb = lo;
    pbe = min(hi, nbc);
    pnc = cn.nc;
    // fused step with an eviction: record cn.nc - 1 is written by the unit's appender
    pwait = (p.fuse && (c.W == 0 || cn.nw == c.W) && cn.nc > 0) ? (cn.nc - 1) / 16 : -1;
    prec = (uint32_t)pu * (uint32_t)c.cap + 16u * (uint32_t)pb;
#if MSTF_UNIFORM
    // (the counters come from global loads: re-assert warp-uniformity of the cursor)
    pb = __shfl_sync(0xffffffffu, pb, 0);
    pbe = __shfl_sync(0xffffffffu, pbe, 0);
    pnc = __shfl_sync(0xffffffffu, pnc, 0);
    pwait = __shfl_sync(0xffffffffu, pwait, 0);
    prec = __shfl_sync(0xffffffffu, prec, 0);
#endif
  };
  p_unit();
  // advance the producer to its next compressed block (or done)
  auto p_advance = [&]() {
    ++pb;
    prec += 16u;
    while (!pdone && pb >= pbe) {
      ++pu;
      if (pu >= c.U || unit_start(p, pu, cpu) >= x1) { pdone = true; break; }
      p_unit();
    }
  };
  // lane 0: TMA of block (pu, pb) into stage pseq % kWNst; pr = its record index, ns = 2 n + stage
  // (passed in so that they can be made provably warp-uniform before the lane-0 branch)
  auto p_issue = [&](uint32_t pr, uint32_t ns) {
    const uint32_t n = ns >> 1;
    if (pb == pwait) {
      // this block holds the record the step's append writes: wait for it (TMA = async proxy)
      wait_ready(p.ready + pu);
      fence_proxy_async_global();
    }
    const uint32_t s = ns & 1u;
    const uint32_t st = wbase + s * (uint32_t)p.stage_bytes, bar = bar0 + 8u * s;
    const uint32_t bytes_bm = n * 16, bytes_k = n * p.rqk, bytes_v = n * p.rqv;
    const uint8_t* g_kbm = reinterpret_cast<const uint8_t*>(c.bm[0]) + (size_t)pr * 16u;
    const uint8_t* g_vbm = reinterpret_cast<const uint8_t*>(c.bm[1]) + (size_t)pr * 16u;
    const uint8_t* g_kv = reinterpret_cast<const uint8_t*>(c.val[0]) + (size_t)pr * (uint32_t)p.rqk;
    const uint8_t* g_vv = reinterpret_cast<const uint8_t*>(c.val[1]) + (size_t)pr * (uint32_t)p.rqv;
    mbar_expect_tx_u32(bar, 2 * bytes_bm + bytes_k + bytes_v);
    bulk_g2s_u32(st, g_kbm, bytes_bm, bar);
    bulk_g2s_u32(st + p.off_kval, g_kv, bytes_k, bar);
    bulk_g2s_u32(st + p.off_vbm, g_vbm, bytes_bm, bar);
    bulk_g2s_u32(st + p.off_vval, g_vv, bytes_v, bar);
  };
  // every lane: the issue of the next block (fence: the stage is being refilled, WAR vs the TMA)
  auto p_issue_warp = [&](bool fence) {
    uint32_t pr = prec, ns = 2u * (uint32_t)min(16, pnc - pb * 16) + (uint32_t)(pseq & (kWNst - 1));
#if MSTF_UNIFORM
    pr = __shfl_sync(0xffffffffu, pr, 0);
    ns = __shfl_sync(0xffffffffu, ns, 0);
#endif
#if MSTF_UNIFORM
    if (elect_one()) {  // (lane 0; an elected lane lets ptxas drop the per-copy uniformity loop)
#else
    if (lane == 0) {
#endif
      if (fence) fence_proxy_async_smem();
      p_issue(pr, ns);
    }
  };
  while (!pdone && pb >= pbe) {  // first unit may hold no compressed block of this range
    ++pu;
    if (pu >= c.U || unit_start(p, pu, cpu) >= x1) { pdone = true; break; }
    p_unit();
  }
  // first stages: issued before this warp's fused appends, except a block that holds a record
  // this step's append writes (its appender may be this warp)
  while (pseq < kPreIssue && !pdone && pb != pwait) {
    p_issue_warp(false);
    ++pseq;
    p_advance();
  }
  fused_appends();
  if (lane == 0) trace_at(P, 1);
  while (pseq < kPreIssue && !pdone) {
    p_issue_warp(false);
    ++pseq;
    p_advance();
  }

  // ---- consumer state. Score product in the transposed form S^T[token][head] (A = K tokens,
  // B = q): lane (g, t) ends with tokens g, g+8 of heads 2t, 2t+1 (c0..c3); for G <= 4 the head
  // columns n are heads n & 3 (duplicated), for G = 8 heads n. movmatrix turns a P^T tile into
  // lane (g, t) = [head column g][tokens 2t, 2t+1], the B operand of the V product, whose
  // columns are (head n & 3 (+4 nt), parity n >> 2).
  constexpr int NT = G8 ? 2 : 1;  // 4-head tiles of the V product
  uint32_t qf[16];                // B operand of the score MMAs: q[head][32t .. 32t+31]
  float acc[NT][4][4];            // O'[pair][(head, parity)] per V n-tile, 4 m-tiles
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // softmax state of heads 2t, 2t+1 (log2 domain)
  const uint32_t par = (uint32_t)(g >> 2);
  const uint32_t sel_lo = par ? 0x1044u : 0x4410u, sel_hi = par ? 0x3244u : 0x4432u;
  // build role of this lane: token lane & 15 of K (lanes 0-15) or V (16-31)
  const uint32_t raw_off = lane < 16 ? (uint32_t)(p.off_kval + (lane & 15) * p.rqk)
                                     : (uint32_t)(p.off_vval + (lane & 15) * p.rqv);
  const uint32_t ydst = lane < 16 ? ypk + 4u * (uint32_t)((lane & 15) * p.swk) : ypv + 4u * (uint32_t)((lane & 15) * p.swv);
  const int nch_me = (lane < 16 ? p.kpk : p.kpv) >> 3;
  const uint32_t bm_off = lane < 16 ? (uint32_t)(16 * (lane & 15)) : (uint32_t)(p.off_vbm + 16 * (lane & 15));
  int qu = -1;
  int cseq = 0;  // compressed blocks consumed

  // a5: S^T (16 tokens x 8 head columns) += K_blk . q^T over the 8 k-steps (two chains)
  auto scores = [&](float (&sc)[4], const uint32_t (&k0)[16], const uint32_t (&k1)[16]) {
    float s2[4] = {0.f, 0.f, 0.f, 0.f};
    sc[0] = sc[1] = sc[2] = sc[3] = 0.f;
#pragma unroll
    for (int s = 0; s < 8; s += 2) {
      mma16816(sc, k0[2 * s], k1[2 * s], k0[2 * s + 1], k1[2 * s + 1], qf[2 * s], qf[2 * s + 1]);
      mma16816(s2, k0[2 * s + 2], k1[2 * s + 2], k0[2 * s + 3], k1[2 * s + 3], qf[2 * s + 2], qf[2 * s + 3]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) sc[i] += s2[i];
  };
  // a7: online softmax over the block (tokens g, g+8 valid: vg, vg8), rescale of the
  // accumulators; bb[nt] = B operand of the V product {k-step 0 lo, hi, k-step 1 lo, hi}
  auto softmax = [&](const float (&sc)[4], bool vg, bool vg8, uint32_t (&bb)[NT][4]) {
    const float x0 = vg ? sc[0] * p.scale_log2 : -INFINITY, x1 = vg ? sc[1] * p.scale_log2 : -INFINITY;
    const float x2 = vg8 ? sc[2] * p.scale_log2 : -INFINITY, x3 = vg8 ? sc[3] * p.scale_log2 : -INFINITY;
    // Lazy rescale: the running reference max m moves only when a score exceeds it by more than
    // p.lazy_log2 = 8 (then P <= 2^8, still rounded to fp16 as always; l and o are fp32, and the
    // combine merges slots by their own m, so any reference value is exact algebra). The common
    // case skips the max reduction and the accumulator rescale. Partials handed to the caller
    // (sequence split) use 0: m is then the exact running max, as the ABI states.
    const bool need = fmaxf(fmaxf(x0, x2) - m0, fmaxf(x1, x3) - m1) > p.lazy_log2;
    if (__any_sync(0xffffffffu, need)) {
      float b0 = fmaxf(x0, x2), b1 = fmaxf(x1, x3);
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        b0 = fmaxf(b0, __shfl_xor_sync(0xffffffffu, b0, o));
        b1 = fmaxf(b1, __shfl_xor_sync(0xffffffffu, b1, o));
      }
      const float n0 = fmaxf(m0, b0), n1 = fmaxf(m1, b1);
      const float a0 = ex2(m0 - n0), a1 = ex2(m1 - n1);
      l0 *= a0;
      l1 *= a1;
      m0 = n0;
      m1 = n1;
      // accumulator columns 2t, 2t+1 of tile nt hold heads (2t & 3) + 4 nt, (2t+1 & 3) + 4 nt
      float aa[NT][2];
      if constexpr (G8) {
        const float o0 = __shfl_xor_sync(0xffffffffu, a0, 2), o1 = __shfl_xor_sync(0xffffffffu, a1, 2);
        aa[0][0] = t < 2 ? a0 : o0; aa[0][1] = t < 2 ? a1 : o1;
        aa[1][0] = t < 2 ? o0 : a0; aa[1][1] = t < 2 ? o1 : a1;
      } else {
        aa[0][0] = a0;
        aa[0][1] = a1;
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[nt][i][0] *= aa[nt][0]; acc[nt][i][1] *= aa[nt][1];
          acc[nt][i][2] *= aa[nt][0]; acc[nt][i][3] *= aa[nt][1];
        }
      }
    }
    const float p0 = ex2(x0 - m0), p1 = ex2(x1 - m1), p2 = ex2(x2 - m0), p3 = ex2(x3 - m1);
    l0 += p0 + p2;
    l1 += p1 + p3;
    // P^T tiles (tokens g / g+8, heads 2t, 2t+1) -> P tiles [head g][tokens 2t, 2t+1 (+8)]
    uint32_t M[2] = {movmatrix_t(pack_half2(p0, p1)), movmatrix_t(pack_half2(p2, p3))};
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      if constexpr (G8) {
        const uint32_t other = __shfl_xor_sync(0xffffffffu, M[ks], 16);
        const uint32_t m_lo = g < 4 ? M[ks] : other, m_hi = g < 4 ? other : M[ks];
        bb[0][2 * ks] = prmt(m_lo, 0u, sel_lo);
        bb[0][2 * ks + 1] = prmt(m_lo, 0u, sel_hi);
        bb[1][2 * ks] = prmt(m_hi, 0u, sel_lo);
        bb[1][2 * ks + 1] = prmt(m_hi, 0u, sel_hi);
      } else {
        bb[0][2 * ks] = prmt(M[ks], 0u, sel_lo);
        bb[0][2 * ks + 1] = prmt(M[ks], 0u, sel_hi);
      }
    }
  };
  // a8 for k-step ks (tokens 8 ks + 2t (va), 8 ks + 2t + 1 (vb)):
  // O'[pair][(head, parity)] += V'[pair][(token, e)] . P'
  auto values_ks = [&](int ks, const uint32_t (&va)[8], const uint32_t (&vb)[8], const uint32_t (&bb)[NT][4]) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
        mma16816(acc[nt][mt], va[mt], va[4 + mt], vb[mt], vb[4 + mt], bb[nt][2 * ks], bb[nt][2 * ks + 1]);
  };

  for (int u = u_first; u < c.U; ++u) {
    const int us = unit_start(p, u, cpu);
    if (us >= x1) break;
    int lo, hi, nbc;
    Counters cn;
    seg_bounds(u, lo, hi, nbc, cn);
    if (lo >= hi) {  // only start-cost units of u in this range: an empty partial (weight 0)
      if (lane < p.G) *reinterpret_cast<float2*>(p.ws_ml + (((size_t)P + u) * p.G + lane) * 2) = make_float2(-INFINITY, 0.f);
      continue;
    }
    if (u != qu) {  // q of the unit: head column g (g & 3 when G <= 4); k-step s: channels
      qu = u;        // 16s + 2t, +1 (qf[2s]) and 16s + 8 + 2t, +1 (qf[2s+1]) -- word 4j + t of slot j
      const int h = G8 ? g : (g & 3);
      if (h < p.G) {
        const uint32_t* qp = reinterpret_cast<const uint32_t*>(p.q + ((size_t)u * p.G + h) * kD) + t;
#pragma unroll
        for (int i = 0; i < 16; ++i) qf[i] = __ldg(qp + 4 * i);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) qf[i] = 0u;
      }
    }
    m0 = m1 = -INFINITY;
    l0 = l1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[nt][i][0] = acc[nt][i][1] = acc[nt][i][2] = acc[nt][i][3] = 0.f;
    if (lane == 0 && hi > nbc && c.W > 0) {  // window rows are read after the unit's records
      l2_prefetch(c.win[0] + (size_t)u * c.W * kD, (uint32_t)c.W * kD * 2);
      l2_prefetch(c.win[1] + (size_t)u * c.W * kD, (uint32_t)c.W * kD * 2);
    }

    // -------- compressed blocks [lo, min(hi, nbc))
    const int bend = min(hi, nbc);
    for (int b = lo; b < bend; ++b, ++cseq) {
      const int s = cseq & (kWNst - 1);
      const uint32_t st = wbase + (uint32_t)(s * p.stage_bytes);
      mbar_wait_u32(bar0 + 8 * s, (uint32_t)(cseq / kWNst) & 1u);
      if (cseq == 0 && lane == 0) trace_at(P, 2);
      if constexpr (kPreIssue < kWNst) {  // top the ring up once the first block has landed
        if (!pdone && pseq < cseq + kWNst) {
          p_issue_warp(false);  // (into the other stage: never used yet)
          ++pseq;
          p_advance();
        }
      }
      const int nvalid = min(16, cn.nc - b * 16);
      // this lane's token's bitmap words (for the pair-entry prefix addresses)
      const bool tok_ok = (lane & 15) < nvalid;
      const uint4 bm_me = MSTF_PREFIX && tok_ok ? lds128(st + bm_off) : make_uint4(0u, 0u, 0u, 0u);
#if MSTF_ZBM
      // a token past the block's end (partial last block): its bitmap slot in the stage holds
      // stale bytes; the token's lane zeroes it, so that every lane below loads bitmaps
      // unconditionally (zero bits: masked gathers, prefix addresses at the row base)
      if (!tok_ok) sts128(st + bm_off, 0u, 0u, 0u, 0u);
#endif
      if constexpr (Q4)
        build_token_q4<NK == NV ? NK : 0>(st + raw_off, ydst, nch_me, bm_me);
      else
        build_token<NK == NV ? NK : 0>(st + raw_off, ydst, nch_me, bm_me);
      // bitmaps (4 words) of K tokens g, g + 8 and V tokens 2t, 2t+1, 8+2t, 9+2t (R5, R6)
      const int tk[4] = {2 * t, 2 * t + 1, 8 + 2 * t, 9 + 2 * t};
#if MSTF_ZBM
      __syncwarp();  // the zeroed slots before the other lanes' loads
      const uint4 kb0 = lds128(st + 16 * g);
      const uint4 kb1 = lds128(st + 16 * (g + 8));
      uint4 vbm[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) vbm[x] = lds128(st + p.off_vbm + 16 * tk[x]);
#else
      const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
      const uint4 kb0 = g < nvalid ? lds128(st + 16 * g) : z4;
      const uint4 kb1 = g + 8 < nvalid ? lds128(st + 16 * (g + 8)) : z4;
      uint4 vbm[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) vbm[x] = tk[x] < nvalid ? lds128(st + p.off_vbm + 16 * tk[x]) : z4;
#endif
      __syncwarp();
      // the stage is fully read: refill it with block cseq + kWNst (WAR vs the TMA write)
      if (!pdone) {
        p_issue_warp(true);
        ++pseq;
        p_advance();
      }
      uint32_t bb[NT][4];
      // a5: S^T += K_blk . q^T, k-step by k-step (two accumulation chains)
      float sc[4];
      {
        TokGather t0, t1;
        tok_prep<(MSTF_PREFIX_SEL & 1) != 0>(t0, kb0, ypk + 4u * (uint32_t)(g * p.swk), 7u - 2u * (uint32_t)t, 4u * (uint32_t)p.kpk);
        tok_prep<(MSTF_PREFIX_SEL & 1) != 0>(t1, kb1, ypk + 4u * (uint32_t)((g + 8) * p.swk), 7u - 2u * (uint32_t)t, 4u * (uint32_t)p.kpk);
        float s2[4] = {0.f, 0.f, 0.f, 0.f};
        sc[0] = sc[1] = sc[2] = sc[3] = 0.f;
#define MSTF_KS(S)                                                                                              \
  mma16816((S & 1) ? s2 : sc, gather_k<2 * S>(t0), gather_k<2 * S>(t1), gather_k<2 * S + 1>(t0), gather_k<2 * S + 1>(t1), \
           qf[2 * S], qf[2 * S + 1]);
        MSTF_KS(0) MSTF_KS(1) MSTF_KS(2) MSTF_KS(3) MSTF_KS(4) MSTF_KS(5) MSTF_KS(6) MSTF_KS(7)
#undef MSTF_KS
#pragma unroll
        for (int i = 0; i < 4; ++i) sc[i] += s2[i];
      }
      // a8, k-step ks: tokens tk[2ks] (va) and tk[2ks+1] (vb); va[mt] / va[4+mt] = rows g / g+8
      auto vgather = [&](int ks, uint32_t (&va)[8], uint32_t (&vb)[8]) {
        TokGather ta, tb;
        const uint32_t sx = 15u - 2u * (uint32_t)g;
        tok_prep<(MSTF_PREFIX_SEL & 2) != 0>(ta, vbm[2 * ks], ypv + 4u * (uint32_t)(tk[2 * ks] * p.swv), sx, 4u * (uint32_t)p.kpv);
        tok_prep<(MSTF_PREFIX_SEL & 2) != 0>(tb, vbm[2 * ks + 1], ypv + 4u * (uint32_t)(tk[2 * ks + 1] * p.swv), sx, 4u * (uint32_t)p.kpv);
        va[0] = gather_v<0, 0>(ta); va[4] = gather_v<0, 1>(ta); vb[0] = gather_v<0, 0>(tb); vb[4] = gather_v<0, 1>(tb);
        va[1] = gather_v<1, 0>(ta); va[5] = gather_v<1, 1>(ta); vb[1] = gather_v<1, 0>(tb); vb[5] = gather_v<1, 1>(tb);
        va[2] = gather_v<2, 0>(ta); va[6] = gather_v<2, 1>(ta); vb[2] = gather_v<2, 0>(tb); vb[6] = gather_v<2, 1>(tb);
        va[3] = gather_v<3, 0>(ta); va[7] = gather_v<3, 1>(ta); vb[3] = gather_v<3, 0>(tb); vb[7] = gather_v<3, 1>(tb);
      };
      // V k-step 0 gathers are issued before the softmax (they do not depend on it), so their
      // shared-memory latency overlaps the shuffles and exp2 of the softmax
      uint32_t va0[8], vb0[8];
      vgather(0, va0, vb0);
      softmax(sc, g < nvalid, g + 8 < nvalid, bb);
      values_ks(0, va0, vb0, bb);
      {
        uint32_t va[8], vb[8];
        vgather(1, va, vb);
        values_ks(1, va, vb, bb);
      }
      __syncwarp();  // every lane's gathers precede the next block's pair-array builds (WAR)
    }

    // -------- window blocks [max(lo, nbc), hi): dense ring rows (a6)
    const int wlo = max(lo, nbc);
    if (wlo < hi) {
      if (p.fuse) {
        if (lane == 0) wait_ready(p.ready + u);
        __syncwarp();
      }
      const int first = c.W > 0 ? cn.nc % c.W : 0;
      const uint16_t* wk = c.win[0] + (size_t)u * c.W * kD;
      const uint16_t* wv = c.win[1] + (size_t)u * c.W * kD;
      for (int x = wlo; x < hi; ++x) {
        const int row0 = (x - nbc) * 16;
        auto ok = [&](int r) {  // ring slot row0 + r holds a window token
          const int slot = row0 + r;
          int age = slot - first;
          if (age < 0) age += c.W;
          return slot < c.W && age < cn.nw;
        };
        if (!__any_sync(0xffffffffu, ok(lane & 15))) continue;
        const int tk[4] = {2 * t, 2 * t + 1, 8 + 2 * t, 9 + 2 * t};
        uint32_t bb[NT][4];
        {
          float sc[4];
          uint32_t kk[2][16];
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const int tok = g + 8 * nt;
            if (ok(tok)) {
              // slot j = 2s + hh: channels 16s + 8hh + 2t, +1 = word 4j + t of the row
              const uint32_t* pp = reinterpret_cast<const uint32_t*>(wk + (size_t)(row0 + tok) * kD) + t;
#pragma unroll
              for (int i = 0; i < 16; ++i) kk[nt][i] = __ldcg(pp + 4 * i);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) kk[nt][i] = 0u;
            }
          }
          scores(sc, kk[0], kk[1]);
          softmax(sc, ok(g), ok(g + 8), bb);
        }
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          uint32_t vv[2][8];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int xx = 2 * ks + e;
            if (ok(tk[xx])) {
              // rows g / g + 8 of m-tile mt: pair 16mt + g / 16mt + 8 + g = word of the row
              const uint32_t* pp = reinterpret_cast<const uint32_t*>(wv + (size_t)(row0 + tk[xx]) * kD) + g;
#pragma unroll
              for (int mt = 0; mt < 4; ++mt) {
                vv[e][mt] = __ldcg(pp + 16 * mt);
                vv[e][4 + mt] = __ldcg(pp + 16 * mt + 8);
              }
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i) vv[e][i] = 0u;
            }
          }
          values_ks(ks, vv[0], vv[1], bb);
        }
      }
    }

    // -------- segment partial (slot P + u): m, l (log2 domain), o unnormalised; cta_merge: the
    // warp's one partial goes to its pair-array region (free after its last block)
    const size_t slot = (size_t)P + u;
    float* dml = p.ws_ml + slot * p.G * 2;
    float* dO = p.ws_o + slot * p.G * kD;
    if (p.cta_merge) {
      dO = reinterpret_cast<float*>(smem + (ypk - smem_u32(smem)));
      dml = dO + p.G * kD;
      if (lane == 0) s_wunit[warp] = u;
    }
    float lt0 = l0, lt1 = l1;
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      lt0 += __shfl_xor_sync(0xffffffffu, lt0, o);
      lt1 += __shfl_xor_sync(0xffffffffu, lt1, o);
    }
    // lanes g = 0: heads 2t, 2t+1 (G <= 4: t < 2 are the real heads; G = 8: every t)
    if (g == 0) {
      if (2 * t < p.G && (G8 || t < 2)) *reinterpret_cast<float2*>(dml + (2 * t) * 2) = make_float2(m0, lt0);
      if (2 * t + 1 < p.G && (G8 || t < 2)) *reinterpret_cast<float2*>(dml + (2 * t + 1) * 2) = make_float2(m1, lt1);
    }
    // accumulators of tile nt: heads hA = 2(t & 1) + 4 nt (c0, c2), hA + 1 (c1, c3), parity t >> 1;
    // rows g: pair 16mt + g (channel 32mt + 2g + par), rows g+8: pair 16mt + 8 + g
    const int pp_ = t >> 1;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int hA = 2 * (t & 1) + 4 * nt;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int h = hA + e;
        if (h < p.G) {
          float* o = dO + h * kD + 2 * g + pp_;
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
            o[32 * mt] = acc[nt][mt][e];
            o[32 * mt + 16] = acc[nt][mt][2 + e];
          }
        }
      }
    }
  }
  }  // x0 < x1
  if (lane == 0) trace_at(P, 3);
  if (p.cta_merge) {
    // merge the CTA's warp partials per unit (shared memory) into one partial (slot CTA + u of ws2)
    __syncthreads();
    const int cb = (int)blockIdx.x, wpc = p.wpc;
    const int X0 = worker_begin(p, S, cb * wpc), X1 = worker_begin(p, S, (cb + 1) * wpc);
    if (X0 < X1) {
      const int uA = unit_of_cost(p, X0, cpu), uB = unit_of_cost(p, X1 - 1, cpu);
      const uint32_t wb = (uint32_t)p.warp_bytes / 4;
      const float* so0 = reinterpret_cast<const float*>(smem + (ypk - smem_u32(smem))) - warp * wb;  // warp 0's
      int wu[kWMaxWarps];  // the unit of each warp's partial (-1: none), in registers
#pragma unroll
      for (int w = 0; w < kWMaxWarps; ++w) wu[w] = w < wpc ? s_wunit[w] : -1;
      for (int u = uA; u <= uB; ++u) {
        for (int i = threadIdx.x; i < p.G * kD; i += blockDim.x) {
          const int h = i / kD;
          // all loads independent (unrolled, selects instead of branches): one smem round trip
          float mw[kWMaxWarps], lw[kWMaxWarps], ow[kWMaxWarps];
#pragma unroll
          for (int w = 0; w < kWMaxWarps; ++w) {
            const float* b2 = so0 + (w < wpc ? w : 0) * wb;
            const float2 ml = *reinterpret_cast<const float2*>(b2 + p.G * kD + 2 * h);
            const bool mine = wu[w] == u;  // other regions may hold pair-array bits: select, not scale
            mw[w] = mine ? ml.x : -INFINITY;
            lw[w] = mine ? ml.y : 0.f;
            ow[w] = mine ? b2[i] : 0.f;
          }
          float mm = -INFINITY;
#pragma unroll
          for (int w = 0; w < kWMaxWarps; ++w) mm = fmaxf(mm, mw[w]);
          float lsum = 0.f, osum = 0.f;
          if (mm != -INFINITY) {
#pragma unroll
            for (int w = 0; w < kWMaxWarps; ++w) {
              const float a = mw[w] == -INFINITY ? 0.f : ex2(mw[w] - mm);  // lw = ow = 0 there
              lsum += a * lw[w];
              osum += a * ow[w];
            }
          }
          const size_t slot = (size_t)cb + u;
          p.ws2_o[slot * p.G * kD + i] = osum;
          if ((i & (kD - 1)) == 0) *reinterpret_cast<float2*>(p.ws2_ml + (slot * p.G + h) * 2) = make_float2(mm, lsum);
        }
      }
    }
    if (lane == 0) trace_at(P, 4);
  }
}

// Ragged caches: cost prefix over the units from the device counters (one CTA).
__global__ void mstf_cost_prefix_kernel(const WParams p) {
  pdl_launch_dependents();
  pdl_wait();
  __shared__ int s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int s_w[32];
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < p.c.U; base += blockDim.x) {
    const int u = base + threadIdx.x;
    const int v = u < p.c.U ? cost_of(p, counters_of(p, u).nc) : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int x = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      s_w[lane] = x;
    }
    __syncthreads();
    const int before = s_carry + (warp ? s_w[warp - 1] : 0);
    if (u < p.c.U) p.pref[u] = before + incl - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry = before + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) p.pref[p.c.U] = s_carry;
}

// a9: one CTA per unit merges the unit's partial slots (the workers overlapping its cost
// range). G warps (one per head) x S sub-warps splitting the slots when units are few.
// In a fused step it then writes the unit's post-append counters and clears its ready flag.
template <bool SUB>
__global__ void __launch_bounds__(512) mstf_warp_combine_kernel(const WParams p) {
  extern __shared__ __align__(16) float s_comb[];
  const int G = p.G;
  const int u = blockIdx.x, wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = SUB ? wi % G : wi, sub = SUB ? wi / G : 0, Sn = SUB ? blockDim.x / (32 * G) : 1;
  // Uniform caches: the partition (S, cost per unit) follows from this unit's own counters, which
  // only this CTA writes (below) and which were last written one decode step ago -- read before
  // the grid-dependency wait, so that the wait is followed directly by the partial loads. This
  // kernel signals its dependents only after its wait: a running combine then implies that
  // every kernel before the attention launch it follows has completed (R-PDL, DESIGN 7.1).
  int nc_u = 0, nw_u = 0, cpu = 0;
  long long S = 0;
  if (p.uniform) {
    nc_u = p.c.n_comp[u];
    nw_u = p.c.n_win[u];
    int nc = nc_u;
    if (p.fuse && (p.c.W == 0 || nw_u == p.c.W)) nc += 1;  // counters_of, from the values just read
    cpu = cost_of(p, nc);
    S = (long long)p.c.U * cpu;
  }
  pdl_wait();  // partials (and the ragged cost prefix) come from the kernels just before
  pdl_launch_dependents();
  if (threadIdx.x == 0) trace_at(65536 + blockIdx.x, 0);
  if (!p.uniform) {
    S = p.hdr[0];
    cpu = p.hdr[1];
  }
  const int us = cpu ? u * cpu : p.pref[u], ue = cpu ? (u + 1) * cpu : p.pref[u + 1];
  // workers overlapping [us, ue): first = owner of us, last = owner of ue - 1
  int wf = worker_of(p, S, us), wl = worker_of(p, S, ue - 1);
  const float* ws_o = p.ws_o;
  const float* ws_ml = p.ws_ml;
  if (p.cta_merge) {  // one partial per CTA (slot CTA + u of ws2)
    wf /= p.wpc;
    wl /= p.wpc;
    ws_o = p.ws2_o;
    ws_ml = p.ws2_ml;
  }
  const int np_ = wl - wf + 1;
  const int i_lo = np_ * sub / Sn, i_hi = np_ * (sub + 1) / Sn;
  float m_max = -INFINITY, l_sum = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (h < G) {
    constexpr int kB = kCombBatch;  // slots per batch: all their loads are issued before any math
    for (int i0 = i_lo; i0 < i_hi; i0 += kB) {
      const int cnt = min(kB, i_hi - i0);
      float2 ml = make_float2(-INFINITY, 0.f);
      if (lane < cnt) ml = *reinterpret_cast<const float2*>(ws_ml + ((size_t)(wf + i0 + lane + u) * G + h) * 2);
      float4 v[kB];
#pragma unroll
      for (int i = 0; i < kB; ++i)
        v[i] = i < cnt ? *(reinterpret_cast<const float4*>(ws_o + ((size_t)(wf + i0 + i + u) * G + h) * kD) + lane)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      float mb = ml.x;
#pragma unroll
      for (int o = 16; o; o >>= 1) mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, o));
      const float mn = fmaxf(m_max, mb);
      if (mn == -INFINITY) continue;
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
        if (wi2 != 0.f) {  // an empty segment's o slot is never written
          acc.x += wi2 * v[i].x; acc.y += wi2 * v[i].y; acc.z += wi2 * v[i].z; acc.w += wi2 * v[i].w;
        }
      }
    }
  }
  if (SUB && Sn > 1) {
    float* s_acc = s_comb;
    float2* s_ml = reinterpret_cast<float2*>(s_comb + (Sn - 1) * G * kD);
    if (sub > 0 && h < G) {
      *reinterpret_cast<float4*>(s_acc + ((sub - 1) * G + h) * kD + 4 * lane) = acc;
      if (lane == 0) s_ml[(sub - 1) * G + h] = make_float2(m_max, l_sum);
    }
    __syncthreads();
    if (sub == 0 && h < G) {
      for (int j = 0; j < Sn - 1; ++j) {
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
  }
  if (sub == 0 && h < G) {
    const size_t oi = ((size_t)u * G + h) * kD + 4 * lane;
    if (p.part_ml) {  // sequence-split shard: unnormalised partials (log2 domain)
      *reinterpret_cast<float4*>(p.part_o + oi) = acc;
      if (lane == 0) *reinterpret_cast<float2*>(p.part_ml + ((size_t)u * G + h) * 2) = make_float2(m_max, l_sum);
    } else {
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
  }
  if (threadIdx.x == 0) trace_at(65536 + blockIdx.x, 1);
  if (p.fuse && threadIdx.x == 0) {  // a4 bookkeeping of the fused step (after every reader)
    const int nc = nc_u, nw = nw_u;  // (fuse implies uniform caches: read before the wait)
    if (p.c.W == 0 || nw == p.c.W) p.c.n_comp[u] = nc + 1; else p.c.n_win[u] = nw + 1;
    p.ready[u] = 0;
  }
}

template <int NK, int NV, bool Q4 = false>
void* pick_kernel(bool g8) {
  return g8 ? (void*)mstf_attn_warp_kernel<NK, NV, true, Q4> : (void*)mstf_attn_warp_kernel<NK, NV, false, Q4>;
}

}  // namespace

// ---------------------------------------------------------------- host side
static size_t r256(size_t b) { return (b + 255) / 256 * 256; }

// cudaFuncSetAttribute once per kernel and size (not per call: keeps the host path short and
// the launch sequence capturable in a CUDA graph after the first, uncaptured, call).
static cudaError_t set_max_smem(void* kern, int bytes) {
  static void* keys[32];
  static int vals[32];
  static int n = 0;
  for (int i = 0; i < n; ++i)
    if (keys[i] == kern) {
      if (vals[i] >= bytes) return cudaSuccess;
      const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      if (e == cudaSuccess) vals[i] = bytes;
      return e;
    }
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && n < 32) {
    keys[n] = kern;
    vals[n] = bytes;
    ++n;
  }
  return e;
}

size_t warp_ws_bytes(int32_t U, int32_t G, int32_t sm_count) {
  const size_t slots = (size_t)sm_count * kWMaxWarps + U + 1, slots2 = (size_t)sm_count + U + 1;
  return r256(kWHdrInts * sizeof(int)) + r256((size_t)U * sizeof(int)) + r256((size_t)(U + 1) * sizeof(int)) +
         r256(slots * G * 2 * sizeof(float)) + r256(slots * G * kD * sizeof(float)) +
         r256(slots2 * G * 2 * sizeof(float)) + slots2 * G * kD * sizeof(float);
}

bool warp_kernel_supported(int32_t G) { return G >= 1 && G <= 8; }

cudaError_t set_dev_trace(void* buf) {
  if (!MSTF_TRACE) return cudaErrorNotSupported;
  unsigned long long* p = static_cast<unsigned long long*>(buf);
  return cudaMemcpyToSymbol(g_mstf_trace, &p, sizeof(p));
}

// words per token: Y[0..kp]; 4 mod 8 for conflict-free 16-byte build stores (MSTF_B128), else 2 mod 4
// with the V region one word off a 32-word boundary (conflict-free 4-byte stores)
static int pair_sw(int kp) { return MSTF_B128 ? kp + 4 : kp + 2; }

int warp_region_bytes(int32_t kpk, int32_t kpv, int32_t rqk, int32_t rqv, int* stage_bytes) {
  const int st = 16 * (16 + rqk) + 16 * (16 + rqv);
  if (stage_bytes) *stage_bytes = st;
  int pairs = (64 * pair_sw(kpk) + 127) / 128 * 128 + (MSTF_B128 ? 0 : 4) + 64 * pair_sw(kpv);
  if (pairs < kWPartBytes) pairs = kWPartBytes;  // the region also holds a warp's partial (cta_merge)
  return (kWNst * st + (pairs + 7) / 8 * 8 + 8 * kWNst + 127) / 128 * 128;
}

WarpPlan plan_warp_attention(int32_t U, int32_t G, int64_t total_cost, int32_t kpk, int32_t kpv, int32_t rqk,
                             int32_t rqv, int32_t sm_count) {
  WarpPlan pl;
  const int wb = warp_region_bytes(kpk, kpv, rqk, rqv, nullptr);
  int wmax = (int)((227 * 1024) / wb);
  const int wcap = G > 4 ? kWMaxWarps / 2 : kWMaxWarps;
  if (wmax > wcap) wmax = wcap;
  if (wmax < 1) wmax = 1;
  // >= ~4 cost units per worker (each worker pays a segment prologue and writes a partial)
  // dev A/B knobs, read once (no per-call environment lookups on the launch path)
  static const int64_t s_qmin = std::getenv("MSTF_QMIN") ? std::max(1, std::atoi(std::getenv("MSTF_QMIN"))) : 4;
  static const int s_wpc = std::getenv("MSTF_WPC") ? std::atoi(std::getenv("MSTF_WPC")) : 0;
  // Small problems (at most one cost unit per warp fills the GPU, G <= 4): one cost unit per
  // warp, warp partials merged per CTA in shared memory (cta_merge). MSTF_CTAMERGE=0: dev A/B.
  static const int s_ctam = std::getenv("MSTF_CTAMERGE") ? std::atoi(std::getenv("MSTF_CTAMERGE")) : 1;
  const bool small = s_ctam != 0 && G <= 4 && total_cost <= (int64_t)sm_count * wmax &&
                     (total_cost + s_qmin - 1) / s_qmin < (int64_t)sm_count * wmax / 2;
  const int64_t qmin = small ? 1 : s_qmin;
  int64_t workers = (total_cost + qmin - 1) / qmin;
  if (workers < 1) workers = 1;
  int grid = sm_count, wpc = wmax;
  if (workers < (int64_t)grid * wmax) {
    wpc = (int)std::max<int64_t>(1, (workers + grid - 1) / grid);
    if (wpc > wmax) wpc = wmax;
    if ((int64_t)grid * wpc > workers) grid = (int)std::max<int64_t>(1, (workers + wpc - 1) / wpc);
  }
  if (s_wpc >= 1 && s_wpc <= wmax) wpc = s_wpc;  // dev A/B: warps per CTA
  pl.grid = grid;
  pl.wpc = wpc;
  pl.cta_merge = small && wpc > 1 && (int64_t)grid * wpc >= total_cost ? 1 : 0;
  pl.warp_bytes = wb;
  pl.smem = wpc * wb;
  return pl;
}

cudaError_t launch_warp_attention(const CacheView& c, const WarpPlan& plan, int32_t G, int32_t uniform, int32_t fuse,
                                  const uint16_t* q, float scale, const uint16_t* k_new, const uint16_t* v_new,
                                  void* out, int32_t out_f16, float* part_ml, float* part_o, void* ws,
                                  int32_t sm_count, cudaStream_t s) {
  WParams p;
  p.c = c;
  p.q = q;
  p.G = G;
  p.scale_log2 = scale * 1.4426950408889634f;
  // lazy rescale (reference max within 8 of the true max) for the normalised output; the exact
  // running max when the caller receives the partials themselves (m = max, the ABI contract)
  p.lazy_log2 = part_ml ? 0.f : 8.f;
  p.np = plan.grid * plan.wpc;
  p.wpc = plan.wpc;
  sk_cost_params(&p.cs, &p.cw);
  p.uniform = uniform;
  p.fuse = fuse;
  p.kpk = c.kpad[0];
  p.kpv = c.kpad[1];
  p.rqk = c.rq[0];
  p.rqv = c.rq[1];
  p.stage_bytes = 0;
  p.warp_bytes = warp_region_bytes(p.kpk, p.kpv, p.rqk, p.rqv, &p.stage_bytes);
  p.off_kval = 256;
  p.off_vbm = p.off_kval + 16 * p.rqk;
  p.off_vval = p.off_vbm + 256;
  p.swk = pair_sw(p.kpk);
  p.swv = pair_sw(p.kpv);
  uint8_t* w = static_cast<uint8_t*>(ws);
  p.hdr = reinterpret_cast<int*>(w);
  w += r256(kWHdrInts * sizeof(int));
  p.ready = reinterpret_cast<int*>(w);
  w += r256((size_t)c.U * sizeof(int));
  p.pref = reinterpret_cast<int*>(w);
  w += r256((size_t)(c.U + 1) * sizeof(int));
  const size_t slots = (size_t)sm_count * kWMaxWarps + c.U + 1;
  p.ws_ml = reinterpret_cast<float*>(w);
  w += r256(slots * G * 2 * sizeof(float));
  p.ws_o = reinterpret_cast<float*>(w);
  w += r256(slots * G * kD * sizeof(float));
  const size_t slots2 = (size_t)sm_count + c.U + 1;
  p.ws2_ml = reinterpret_cast<float*>(w);
  w += r256(slots2 * G * 2 * sizeof(float));
  p.ws2_o = reinterpret_cast<float*>(w);
  p.cta_merge = plan.cta_merge;
  p.k_new = k_new;
  p.v_new = v_new;
  p.out = out;
  p.out_f16 = out_f16;
  p.part_ml = part_ml;
  p.part_o = part_o;

  cudaError_t e;
  if (!uniform) {
    e = launch_pdl(mstf_cost_prefix_kernel, dim3(1), dim3(1024), 0, s, p);
    if (e != cudaSuccess) return e;
  }
  const bool g8 = G > 4;
  void* kern = nullptr;
  const int nk = c.kpad[0] / 8, nv = c.kpad[1] / 8;
  if (c.vbits == 4) {
    if (nk == nv && nk == 5) kern = pick_kernel<5, 5, true>(g8);
    else if (nk == nv && nk == 8) kern = pick_kernel<8, 8, true>(g8);
    else kern = pick_kernel<0, 0, true>(g8);
  } else if (nk == nv && nk == 5) kern = pick_kernel<5, 5>(g8);
  else if (nk == nv && nk == 8) kern = pick_kernel<8, 8>(g8);
  else if (nk == nv && nk == 4) kern = pick_kernel<4, 4>(g8);
  else if (nk == nv && nk == 2) kern = pick_kernel<2, 2>(g8);
  else kern = pick_kernel<0, 0>(g8);
  void (*kf)(WParams) = reinterpret_cast<void (*)(WParams)>(kern);
  e = set_max_smem(kern, plan.smem);
  if (e != cudaSuccess) return e;
  e = launch_pdl(kf, dim3(plan.grid), dim3(32 * plan.wpc), (size_t)plan.smem, s, p);
  if (e != cudaSuccess) return e;
  // combine: sub-warps per head when a unit has many partial slots (few units)
  const int64_t slots_per_unit = ((int64_t)(p.cta_merge ? plan.grid : p.np) + c.U - 1) / c.U + 2;
  int sub = (int)((slots_per_unit + kCombBatch - 1) / kCombBatch);
  // dev A/B knob (read once): cap on the sub-warps per head
  static const int s_subcap = std::getenv("MSTF_COMBSUB_MAX") ? std::max(1, std::atoi(std::getenv("MSTF_COMBSUB_MAX"))) : 4;
  sub = std::max(1, std::min(std::min(sub, s_subcap), 512 / (32 * G)));
  if (sub == 1) return launch_pdl(mstf_warp_combine_kernel<false>, dim3(c.U), dim3(32 * G), 0, s, p);
  const size_t csmem = (size_t)(sub - 1) * G * (kD * sizeof(float) + sizeof(float2));
  return launch_pdl(mstf_warp_combine_kernel<true>, dim3(c.U), dim3(32 * G * sub), csmem, s, p);
}

}  // namespace mstf
