// kernels.cuh -- launch interfaces shared between the ABI layer (abi.cu) and the
// kernels (compress.cu, attn_warp.cu, dense.cu). Not part of the public ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cstdlib>
#include <utility>

namespace mstf {

// Launch with programmatic stream serialization (PDL): the kernel may start while its
// predecessor in the stream drains; it must pdl_wait() before touching dependent memory.
inline bool pdl_enabled() {  // MSTF_NOPDL=1 (dev): ordinary launches, e.g. for profiler timelines
  static const bool on = std::getenv("MSTF_NOPDL") == nullptr;
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

constexpr int kD = 128;          // head_dim supported by the v1 kernels
constexpr int kTiles = kD / 64;  // 64-bit bitmap words per token record
constexpr int kConsumerWarps = 4; // warps per CTA of the dense baseline kernel
constexpr int kMaxGroup = 8;     // query heads per unit (mma N = 8)
constexpr int kValuesGuard = 16; // bytes after each VALUES buffer (read past the last record, never used)

// Device view of one cache (one tensor = K or V shares the same layout).
struct CacheView {
  uint64_t* bm[2];      // [U][cap][kTiles]
  uint16_t* val[2];     // [U][cap][kpad] fp16 values, or [U][cap][rq] bytes (4-bit payload)
  uint32_t* off[2];     // [U][cap][kTiles]
  uint16_t* win[2];     // [U][max(W,1)][kD]
  int32_t* n_comp;      // [U]
  int32_t* n_win;       // [U]
  int32_t U, W, cap;
  int32_t keep[2], kpad[2];
  int32_t vbits;        // 16: fp16 values; 4: quantized records (NEXT-4)
  int32_t rq[2];        // bytes of one token's value record: 2*kpad (fp16) or the 4-bit record
  const float* kw;      // [U][kD] float32 K channel weights (output-aware pruning), or null
};

cudaError_t launch_set_counters(const CacheView& c, const int32_t* nc_host, const int32_t* nw_host,
                                int32_t uniform_T, cudaStream_t s);
cudaError_t launch_prefill(const CacheView& c, const uint16_t* k, const uint16_t* v, int32_t T,
                           cudaStream_t s);
cudaError_t launch_query_abs_sum(const uint16_t* q, int32_t U, int32_t R, int32_t G, int32_t d, float* w,
                                 cudaStream_t s);
cudaError_t launch_append(const CacheView& c, const uint16_t* k_new, const uint16_t* v_new,
                          cudaStream_t s);

// Stream-K partition cost of one unit (see attn_warp.cu) and its parameters.
int32_t sk_unit_cost(int32_t n_comp, int32_t W);
void sk_cost_params(int32_t* cs, int32_t* cw);
// Sequence split (NEXT-3): partials of an empty shard (m = -inf, l = 0, o = 0), n = U * G.
cudaError_t launch_empty_partials(float* ml, float* o, int32_t n, cudaStream_t s);
// Sequence split (NEXT-3): merge n shards' partials [n][U][G] into O [U][G][kD].
cudaError_t launch_merge_partials(int32_t n, int32_t U, int32_t G, const float* ml, const float* o, void* out,
                                  int32_t out_f16, cudaStream_t s);

// Dense-KV baseline (dense.cu): grid (splits, U) + combine; workspace bytes for `splits`.
size_t dense_ws_bytes(int32_t U, int32_t G, int32_t splits);
cudaError_t launch_dense_attention(const uint16_t* k, const uint16_t* v, const int32_t* lengths, int32_t U,
                                   int32_t G, int32_t t_max, int32_t splits, const uint16_t* q, float scale,
                                   void* out, int32_t out_f16, void* ws, cudaStream_t s);

// r2 attention (attn_warp.cu): one self-contained warp per stream-K worker, TMA-staged blocks,
// device-side partition from the device counters (CUDA-graph replayable), optional fused append.
struct WarpPlan {
  int32_t grid;        // CTAs (<= SMs, one per SM)
  int32_t wpc;         // warps (workers) per CTA
  int32_t cta_merge;   // small problems: warp partials merged per CTA in shared memory
  int32_t warp_bytes;  // shared memory per warp
  int32_t smem;        // dynamic shared memory per CTA
};
bool warp_kernel_supported(int32_t G);
cudaError_t set_dev_trace(void* buf);  // development: per-worker phase stamps (null: off)
size_t warp_ws_bytes(int32_t U, int32_t G, int32_t sm_count);
int warp_region_bytes(int32_t kpk, int32_t kpv, int32_t rqk, int32_t rqv, int* stage_bytes);
WarpPlan plan_warp_attention(int32_t U, int32_t G, int64_t total_cost, int32_t kpk, int32_t kpv, int32_t rqk,
                             int32_t rqv, int32_t sm_count);
// uniform: every unit has the same counters (fuse requires it). fuse: k_new / v_new are appended
// inside the launch (the counters are then advanced by the combine kernel).
cudaError_t launch_warp_attention(const CacheView& c, const WarpPlan& plan, int32_t G, int32_t uniform, int32_t fuse,
                                  const uint16_t* q, float scale, const uint16_t* k_new, const uint16_t* v_new,
                                  void* out, int32_t out_f16, float* part_ml, float* part_o, void* ws,
                                  int32_t sm_count, cudaStream_t s);

// dev: read-only HBM stream over [src, src + bytes) (bench.py's read-peak measurement)
cudaError_t launch_dev_read(const void* src, size_t bytes, uint32_t* sink, int sm_count, cudaStream_t s);


}  // namespace mstf
