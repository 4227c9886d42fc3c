/*
 * mustafar.h -- C ABI of the B200 (sm_100a) Mustafar hot path.
 *
 * Mustafar (arXiv 2505.22913) prunes every token's Key and Value head vector to
 * unstructured sparsity by magnitude, stores the survivors in a bitmap-based sparse
 * format, and computes decode attention directly on that compressed cache.
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, R# = DESIGN.md "Readings".
 *
 * The three calls of the paper's problem statement:
 *   mstf_prune_compress_kv        "KV cache generated in prefill stage is pruned and
 *                                  compressed before the start of decode stage"
 *   mstf_append_token             "KV cache generated in decode stage is kept as-is (dense)
 *                                  while it is within the local window, then pruned and
 *                                  compressed afterwards"
 *   mstf_sparse_decode_attention  Algorithm 1: dense local-window MV + SpMV over
 *                                  the compressed cache, one softmax over the concatenation.
 * plus the dense-KV decode baseline mstf_dense_decode_attention (the comparison the
 * paper's Fig. 5a / Fig. 6 make against dense attention).
 *
 * Conventions (all calls):
 *   - extern "C", no exceptions cross the boundary; every call returns an mstf_status
 *     (0 = OK, < 0 = error) and validates all host-side arguments BEFORE any launch.
 *   - Tensor pointers are DEVICE pointers owned by the caller (e.g. allocated by torch);
 *     the library never allocates or frees device memory and never synchronizes.
 *     `stream` is a cudaStream_t (passed as void*); work is enqueued on it in order.
 *   - fp16 means IEEE binary16 bit patterns; all arrays are dense row-major (C order).
 *   - A "unit" is one (batch, kv-head) pair: U = batch * num_kv_heads, b-major
 *     (u = b * num_kv_heads + h_kv). G = num_q_heads / num_kv_heads query heads share a
 *     unit (GQA; query head h_q maps to h_kv = floor(h_q / G), R11), so the query /
 *     output tensor [batch][num_q_heads][d] is the same memory as [U][G][d].
 *   - One cache handle per stream (single writer).
 */
#ifndef MUSTAFAR_H
#define MUSTAFAR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status codes */
typedef enum {
  MSTF_OK = 0,
  MSTF_EINVAL = -1,     /* null pointer, negative size, bad enum                        */
  MSTF_ESHAPE = -2,     /* head_dim % 64 != 0, num_q_heads % num_kv_heads != 0, T < 0   */
  MSTF_EKEEP = -3,      /* keep_k / keep_v outside [1, head_dim]                        */
  MSTF_ECAPACITY = -4,  /* compressed tokens of some unit would exceed `capacity`       */
  MSTF_EEMPTY = -5,     /* attention requested while some unit holds 0 tokens           */
  MSTF_ECUDA = -6,      /* a CUDA launch/runtime error (cudaGetLastError after launch)  */
  MSTF_ENOTSUP = -7,    /* valid but unsupported here (v1 kernels: head_dim == 128, G<=8)*/
  MSTF_EWORKSPACE = -8  /* workspace pointer null / too small                          */
} mstf_status;

/* ------------------------------------------------------------------ configuration */
typedef struct {
  int32_t batch;         /* B >= 1                                                        */
  int32_t num_q_heads;   /* Hq >= 1, multiple of num_kv_heads                             */
  int32_t num_kv_heads;  /* Hkv >= 1                                                      */
  int32_t head_dim;      /* d, multiple of 64 (1x64 tiles); kernels: d == 128      */
  int32_t keep_k;        /* channels kept per Key token, 1..d   (k = d - floor(s*d), R1)  */
  int32_t keep_v;        /* channels kept per Value token, 1..d (K_s != V_s allowed)*/
  int32_t window;        /* dense local window W >= 0 (paper: 32)                    */
  int32_t capacity;      /* max compressed tokens per unit (records per unit)             */
  int32_t value_bits;    /* payload of the kept values: 16 (or 0) = fp16 values; 4 = the
                            prune-then-quantize payload ("we first
                            prune each token's KV cache before quantization is performed",
                            KIVI 4-bit of tab:joint_quant): per token 4-bit codes with an fp16
                            scale and zero point over its kept values (R25-R27)              */
} mstf_config;

/* k = d - floor(s*d) for s in [0,1) (R1). Returns MSTF_EKEEP for s outside. */
int32_t mstf_keep_from_sparsity(double sparsity, int32_t head_dim);

/* Packed-value slots per token: ceil(k/8)*8 ("multiples-of-8 padding"; R7). */
int32_t mstf_k_pad(int32_t keep);

/* Bytes of one token's value record: 2 * mstf_k_pad(keep) for value_bits 16 (or 0);
 * for value_bits 4, round_up(4 + ceil(keep / 2), 16) (R26). MSTF_EINVAL for other value_bits. */
int32_t mstf_value_record_bytes(int32_t keep, int32_t value_bits);

/* ------------------------------------------------------------------ cache buffers
 * The compressed format ("compressed tiles corresponding to a 1x64 column of the
 * pruned cache. Per-tile bitmap of 64 bits is used to represent the position of
 * non-zeros, and tile offset is used to address the correct position of each tile's
 * starting non-zero"), in the build's per-token record layout (R4-R8):
 *   token p of unit u, once it has left the window, is record p of that unit;
 *   BITMAP_x  u64 [U][capacity][d/64]  bit i of word j <=> channel 64j+i kept (LSB first);
 *                                       exactly keep_x bits set per record (R4)
 *   VALUES_x  u16 [U][capacity][kpad]   kept fp16 bit patterns in ascending channel order,
 *                                       then 0x0000 up to kpad = mstf_k_pad(keep_x) (R6, R7);
 *                                       the buffer is 16 bytes longer (tail guard);
 *             value_bits 4: u8 [U][capacity][rq], rq = mstf_value_record_bytes(keep_x, 4):
 *                                       bytes 0-1 scale (fp16), 2-3 zero point (fp16), byte 4 + i/2
 *                                       the 4-bit code of kept value i (channel order, low nibble
 *                                       for even i), then 0x00 padding; value i reconstructs to
 *                                       f16(code_i * scale + zero) (R25-R27)
 *   OFFSETS_x u32 [U][capacity][d/64]   p*kpad + (kept channels in tiles < j): element index
 *                                       of tile j's first value in the unit's value array (R8)
 *   WIN_x     u16 [U][max(W,1)][d]      dense window ring: token p sits in slot p % W (R9)
 *   N_COMP    i32 [U]                   compressed tokens per unit (device counter)
 *   N_WIN     i32 [U]                   window tokens per unit, <= W (device counter)
 * Every buffer must be 16-byte aligned. Only N_COMP / N_WIN need initialising: to zero
 * (an empty cache, matching the handle's host mirror) unless the first call on the cache
 * is mstf_prune_compress_kv, which writes them. Byte sizes: mstf_cache_buffer_bytes.    */
enum {
  MSTF_BUF_BITMAP_K = 0, MSTF_BUF_BITMAP_V, MSTF_BUF_VALUES_K, MSTF_BUF_VALUES_V,
  MSTF_BUF_OFFSETS_K, MSTF_BUF_OFFSETS_V, MSTF_BUF_WIN_K, MSTF_BUF_WIN_V,
  MSTF_BUF_N_COMP, MSTF_BUF_N_WIN, MSTF_NUM_BUFFERS
};

/* Host-only. Fills sizes[MSTF_NUM_BUFFERS] (bytes). Validates the config. */
int mstf_cache_buffer_bytes(const mstf_config* cfg, size_t sizes[MSTF_NUM_BUFFERS]);

/* Opaque HOST handle: a copy of the config, the caller's device pointers and an exact
 * host mirror of n_comp / n_win (the cache operations are deterministic, so the mirror
 * lets capacity overflow be detected without a device sync). */
typedef struct mstf_cache mstf_cache;

/* buffers[i]: device pointer of buffer i (sizes from mstf_cache_buffer_bytes). *out gets
 * a new handle (host malloc). The handle starts empty (n_comp = n_win = 0 on the mirror;
 * the device counters are written by the first mstf_prune_compress_kv). */
int mstf_cache_create(const mstf_config* cfg, void* const buffers[MSTF_NUM_BUFFERS],
                      mstf_cache** out);
/* Frees the host handle only (device buffers belong to the caller). NULL is a no-op. */
int mstf_cache_destroy(mstf_cache* cache);
/* Host mirror of the per-unit counters (n_comp, n_win may be NULL). No device access. */
int mstf_cache_counts(const mstf_cache* cache, int32_t* n_comp, int32_t* n_win);

/* ------------------------------------------------------------------ prefill ingest
 * Resets the cache and ingests a prefill (A10). k, v: fp16 [U][T][d] device.
 * lengths: optional HOST int32 [U] with 0 <= lengths[u] <= T (ragged prompts; NULL means
 * every unit holds T tokens). For unit u with L = lengths[u]: tokens 0..L-W-1 are pruned
 * (per-token magnitude top-keep, lower channel index pruned first on ties: P:62, P:173,
 * R2, R3) and compressed into records 0..L-W-1; the last min(L, W) tokens are copied
 * dense into the window ring (R9). Errors: ESHAPE (T < 0), EINVAL (lengths out of range),
 * ECAPACITY (L - min(L,W) > capacity for some u), ECUDA.                              */
int mstf_prune_compress_kv(mstf_cache* cache, const void* k, const void* v, int32_t T,
                           const int32_t* lengths, void* stream);

/* ------------------------------------------------------------------ decode append
 * Appends one decode token per unit (A11). k_new, v_new: fp16 [U][d] device
 * (== [batch][num_kv_heads][d]). If a unit's window is full (n_win == W) its oldest window
 * token (position n_comp) is pruned + compressed into record n_comp and n_comp += 1; the
 * new token then takes the freed slot. With W == 0 the new token is compressed directly.
 * Device counters are updated on the device (no host sync; CUDA-graph capturable).
 * Errors: ECAPACITY (host mirror would exceed capacity), ECUDA.                       */
int mstf_append_token(mstf_cache* cache, const void* k_new, const void* v_new, void* stream);

/* ------------------------------------------------------------------ decode attention
 * Algorithm 1 for every unit and each of its G query heads:
 *   S_C = scale * q K_C^T, S_L = scale * q K_L^T, S = softmax(concat(S_C, S_L)),
 *   O = S_C V_C + S_L V_L      (K_C, V_C: compressed tokens; K_L, V_L: window tokens).
 * q: fp16 [U][G][d] device. scale: e.g. 1/sqrt(d) (R10; 1.0 gives the literal Alg. 1).
 * out: device, [U][G][d] float32 (out_dtype = MSTF_OUT_F32) or fp16 (MSTF_OUT_F16).
 * workspace: device scratch of >= mstf_workspace_bytes(cache) bytes (split partials and per-unit
 *            arrival tickets); it must be zero-filled once before its first use -- every call
 *            leaves the tickets at zero again. One workspace per concurrently running call.
 * Split-sequence (flash-decoding) over the compressed tokens; fp16 x fp16 products with
 * fp32 accumulation; softmax in fp32; the softmax weights enter P.V as fp16.
 * Errors: EEMPTY (some unit holds no token), EWORKSPACE, ENOTSUP, ECUDA.               */
enum { MSTF_OUT_F32 = 0, MSTF_OUT_F16 = 1 };
size_t mstf_workspace_bytes(const mstf_cache* cache);
int mstf_sparse_decode_attention(const mstf_cache* cache, const void* q, float scale,
                                 void* out, int32_t out_dtype, void* workspace,
                                 size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------ dense baseline
 * Dense-KV decode attention with the same kernel skeleton (no pruning): the baseline the
 * paper compares against (P:439 cuBLAS batched MV, P:458 FlashAttention-2).
 * k, v: fp16 [U][T_max][d] device; lengths: DEVICE int32 [U] (tokens of each unit, >= 1);
 * q / out / workspace as above (workspace >= mstf_dense_workspace_bytes).               */
size_t mstf_dense_workspace_bytes(int32_t units, int32_t group, int32_t head_dim,
                                  int32_t t_max);
int mstf_dense_decode_attention(const void* k, const void* v, const int32_t* lengths,
                                int32_t units, int32_t group, int32_t head_dim,
                                int32_t t_max, const void* q, float scale, void* out,
                                int32_t out_dtype, void* workspace, size_t workspace_bytes,
                                void* stream);

/* ------------------------------------------------------------------ multi-GPU
 * Contiguous unit range [u0, u1) of rank `rank` among `world`: units are
 * independent, so a shard is just a cache over its U/world units, and its q / out
 * slices are contiguous in [B][Hq][d]. Host-only.                                      */
int mstf_shard_units(int32_t units, int32_t world, int32_t rank, int32_t* u0, int32_t* u1);

/* One decode step of a layer: exactly mstf_append_token(k_new, v_new) followed by
 * mstf_sparse_decode_attention(q, ...) (R12: the new token attends to itself), with the same
 * arguments, layouts, results and errors. P:234 (compress on exit from the window) + Alg. 1.
 * When every unit has the same counters and k_pad selects the register-staged kernel, the
 * append runs inside the attention launch (one kernel + the split combine instead of three
 * launches); otherwise the two calls are made in sequence. The workspace must come from
 * mstf_workspace_bytes, be zero-filled once before first use (it carries per-unit ready flags
 * stamped per call), and not be shared by calls that may run concurrently. */
int mstf_decode_step(mstf_cache* cache, const void* k_new, const void* v_new, const void* q, float scale,
                     void* out, int32_t out_dtype, void* workspace, size_t workspace_bytes, void* stream);

/* Kernels one mstf_decode_step call on this cache (in its current state) launches: 2 fused,
 * 3 unfused; negative status for a NULL handle. Host-only. */
int mstf_decode_step_kernel_count(const mstf_cache* cache);

/* CUDA-graph replay of decode steps (NEXT-1). On a uniform cache (every unit with the same
 * counters) mstf_decode_step's launches take no argument that depends on the counters: the
 * kernels read n_comp / n_win from the device, the fused append's flags are cleared by the
 * step's own combine kernel and the combine advances the device counters. A graph captured
 * around n_layers x mstf_decode_step therefore replays correctly step after step, but the
 * replays bypass the handle, so its host mirror no longer follows the device.
 * mstf_graph_step_check: returns MSTF_OK if `steps` more uniform decode steps fit (every
 *   unit's compressed capacity), MSTF_ECAPACITY if not, MSTF_EINVAL if the cache is not uniform
 *   (a captured step would not be the fused, counter-independent one). Host-only.
 * mstf_graph_step_commit: advances the host mirror by `steps` decode steps that graph replays
 *   enqueued (same rule as mstf_append_token: the oldest window token is compressed once the
 *   window is full). Validates like the check first; host-only, no device access.          */
int mstf_graph_step_check(const mstf_cache* cache, int32_t steps);
int mstf_graph_step_commit(mstf_cache* cache, int32_t steps);

/* Number of kernels one mstf_sparse_decode_attention call on this cache launches (the
 * attention kernel and the split combine), or a negative status for a NULL handle.
 * Host-only; lets callers count launches. */
int mstf_attention_kernel_count(const mstf_cache* cache);

/* ------------------------------------------------------------------ sequence split (NEXT-3)
 * Batch-1 long context has too few units to shard by unit (fewer thread blocks than SMs
 * at batch 1), so the tokens of every unit are split across ranks instead:
 * mstf_seq_split: rank r's prompt tokens [t0, t1) of T. The C = T - min(T, W) tokens that are
 * compressed at prefill are split evenly; the last rank also takes the last min(T, W) tokens (the
 * dense window, R9), so it alone holds a window (W) and takes every decode append; the other
 * ranks build their caches with window 0. The union of the shards is exactly the single-device
 * cache (pruning is per token). Host-only.                                                   */
int mstf_seq_split(int32_t T, int32_t window, int32_t world, int32_t rank, int32_t* t0, int32_t* t1);

/* Algorithm 1 over this cache's tokens only, stopping before the final normalisation: the
 * shard's softmax partials (the a9 combine state of flash-decoding), float32 DEVICE:
 *   ml [U][G][2]: m = max_t s_t*log2(e), l = sum_t 2^(s_t*log2(e) - m);  o [U][G][d]:
 *   o = sum_t 2^(s_t*log2(e) - m) * v_t (not divided by l), s_t = scale * q . k_t.
 * q, scale, workspace as in mstf_sparse_decode_attention. ml 8-byte aligned, o 16-byte aligned.
 * A cache in which EVERY unit is empty (a rank that holds no token, e.g. T < world) writes the
 * merge identity m = -inf, l = 0, o = 0; some-but-not-all units empty is EEMPTY.
 * Errors: as mstf_sparse_decode_attention.                                                     */
int mstf_sparse_decode_attention_partial(const mstf_cache* cache, const void* q, float scale, float* ml,
                                         float* o, void* workspace, size_t workspace_bytes, void* stream);

/* Merge n shards' partials (e.g. all-gathered across ranks) into the attention output:
 *   M = max_i m_i,  O = sum_i 2^(m_i - M) o_i / sum_i 2^(m_i - M) l_i       (the a9 combine)
 * ml: float32 DEVICE [n][units][group][2], o: [n][units][group][head_dim]; out: [units][group]
 * [head_dim] float32 or fp16 (out_dtype). A shard without tokens (m = -inf) contributes nothing;
 * a (unit, head) with no token in any shard gives 0. Errors: EINVAL, ENOTSUP (head_dim != 128,
 * group > 8), ECUDA.                                                                            */
int mstf_merge_partials(int32_t n, int32_t units, int32_t group, int32_t head_dim, const float* ml,
                        const float* o, void* out, int32_t out_dtype, void* stream);

/* ------------------------------------------------------------------ output-aware Key pruning
 * Per-token OUTPUT-AWARE pruning of the Key cache:
 *   S = |K| (.) broadcast(w),  w = sum over the window's queries t of |Q_t|, summed over the
 *   GQA group's query heads.
 * mstf_set_key_weights: every later K compression of this cache (mstf_prune_compress_kv,
 * the evictions of mstf_append_token / mstf_decode_step) keeps, per token, the keep_k channels
 * with the largest score fl32(|k_c| * w[u][c]) (one float32 multiply, round to nearest, R20),
 * lower channel index pruned first on equal scores (R2). V stays magnitude pruned.
 * w: DEVICE float32 [U][head_dim], 16-byte aligned, finite and >= 0, owned by the caller and
 * read by the kernels at run time (update it in stream order between steps); NULL restores
 * magnitude pruning. Errors: EINVAL (misaligned).                                       */
int mstf_set_key_weights(mstf_cache* cache, const float* w);

/* The accumulator of P:86 ("the element-wise L1 accumulation of the current and next 31
 * Query vector"): w[u][c] = sum_{r < R} sum_{g < G} |q[u][r][g][c]| in float32, added in the
 * order r ascending, then g ascending (R21). q: fp16 DEVICE [U][R][G][d] (the window's R
 * queries of each unit's G query heads, in any fixed slot order, e.g. a ring); w: DEVICE
 * float32 [U][d]. R = 0 gives zeros. Errors: EINVAL (null, negative sizes), ECUDA.          */
int mstf_query_abs_sum(const void* q, int32_t units, int32_t slots, int32_t group, int32_t head_dim,
                       float* w, void* stream);

/* Development only (bench.py's read-only roofline denominator), not part of the hot path:
 * streams [src, src + bytes) once with 16-byte loads and nothing else (bytes rounded down to a
 * multiple of 16). src: DEVICE, 16-byte aligned; sink: DEVICE u32 (written only on an
 * impossible XOR pattern, it keeps the loads alive). Asynchronous on `stream`.
 * Errors: EINVAL (null / misaligned), ECUDA.                                                 */
int mstf_dev_read_bandwidth(const void* src, size_t bytes, void* sink, void* stream);

/* Development only: buf (DEVICE u64, or NULL to switch off) receives global-timer stamps (ns)
 * of the attention kernel's phases: [worker][8] with worker = CTA * warps-per-CTA + warp (0:
 * start, 1: after the fused appends, 2: first compressed block landed, 3: done) and, from index
 * 65536, [combine CTA][8] (0: start, 1: done). The caller sizes buf (>= 65536 + U entries x 8)
 * and keeps it alive while set. Only builds with -DMSTF_TRACE=1 record (the stamps are compiled
 * out otherwise). Errors: ENOTSUP (not a trace build), ECUDA.                                */
int mstf_dev_trace(void* buf);

/* Human-readable status (static string). */
const char* mstf_status_string(int32_t status);

/* Library/kernels build identification (static string), e.g. "sm_100a". */
const char* mstf_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* MUSTAFAR_H */
