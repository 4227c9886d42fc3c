// abi.cu -- the extern "C" boundary declared in include/mustafar.h: host-side validation,
// buffer sizing, the exact host mirror of the per-unit counters, and kernel launches.
// No device allocation, no synchronisation.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/mustafar.h"
#include "kernels.cuh"

using namespace mstf;

struct mstf_cache {
  mstf_config cfg;
  CacheView view;
  std::vector<int32_t> nc, nw;  // exact host mirror of n_comp / n_win
};

namespace {

int validate(const mstf_config* c) {
  if (!c) return MSTF_EINVAL;
  if (c->batch < 1 || c->num_q_heads < 1 || c->num_kv_heads < 1 || c->head_dim < 1 || c->window < 0 ||
      c->capacity < 0)
    return MSTF_EINVAL;
  if (c->head_dim % 64 != 0 || c->num_q_heads % c->num_kv_heads != 0) return MSTF_ESHAPE;
  if (c->keep_k < 1 || c->keep_k > c->head_dim || c->keep_v < 1 || c->keep_v > c->head_dim) return MSTF_EKEEP;
  if (c->value_bits != 0 && c->value_bits != 16 && c->value_bits != 4) return MSTF_EINVAL;
  if (c->head_dim != kD || c->num_q_heads / c->num_kv_heads > kMaxGroup) return MSTF_ENOTSUP;
  return MSTF_OK;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline bool aligned8(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 7u) == 0; }
// The combine kernels store 4 outputs per lane: one float4 (f32) or two half2 (f16, 8 bytes).
inline bool out_aligned(const void* out, int32_t out_dtype) {
  return out_dtype == MSTF_OUT_F16 ? aligned8(out) : aligned16(out);
}

}  // namespace

extern "C" {

int32_t mstf_keep_from_sparsity(double s, int32_t d) {
  if (!(s >= 0.0 && s < 1.0) || d < 1) return MSTF_EKEEP;
  return (int32_t)(d - (int32_t)std::floor(s * d));
}

int32_t mstf_k_pad(int32_t keep) { return ((keep + 7) / 8) * 8; }

int32_t mstf_value_record_bytes(int32_t keep, int32_t value_bits) {
  if (keep < 1) return MSTF_EKEEP;
  if (value_bits == 0 || value_bits == 16) return 2 * mstf_k_pad(keep);
  if (value_bits == 4) return ((4 + (keep + 1) / 2 + 15) / 16) * 16;
  return MSTF_EINVAL;
}

int mstf_cache_buffer_bytes(const mstf_config* c, size_t sizes[MSTF_NUM_BUFFERS]) {
  const int st = validate(c);
  if (st != MSTF_OK && st != MSTF_ENOTSUP) return st;
  if (!sizes) return MSTF_EINVAL;
  const size_t U = (size_t)c->batch * c->num_kv_heads, cap = c->capacity, nt = c->head_dim / 64;
  const size_t W = c->window > 0 ? c->window : 1;
  sizes[MSTF_BUF_BITMAP_K] = sizes[MSTF_BUF_BITMAP_V] = U * cap * nt * 8;
  // + kValuesGuard: the attention kernels' per-token loads may read up to 8 bytes past a record
  sizes[MSTF_BUF_VALUES_K] = U * cap * (size_t)mstf_value_record_bytes(c->keep_k, c->value_bits) + kValuesGuard;
  sizes[MSTF_BUF_VALUES_V] = U * cap * (size_t)mstf_value_record_bytes(c->keep_v, c->value_bits) + kValuesGuard;
  sizes[MSTF_BUF_OFFSETS_K] = sizes[MSTF_BUF_OFFSETS_V] = U * cap * nt * 4;
  sizes[MSTF_BUF_WIN_K] = sizes[MSTF_BUF_WIN_V] = U * W * c->head_dim * 2;
  sizes[MSTF_BUF_N_COMP] = sizes[MSTF_BUF_N_WIN] = U * 4;
  return st;
}

int mstf_cache_create(const mstf_config* c, void* const buffers[MSTF_NUM_BUFFERS], mstf_cache** out) {
  const int st = validate(c);
  if (st != MSTF_OK) return st;
  if (!buffers || !out) return MSTF_EINVAL;
  for (int i = 0; i < MSTF_NUM_BUFFERS; ++i)
    if (!buffers[i] || !aligned16(buffers[i])) return MSTF_EINVAL;
  mstf_cache* h = new (std::nothrow) mstf_cache();
  if (!h) return MSTF_EINVAL;
  h->cfg = *c;
  CacheView& v = h->view;
  for (int x = 0; x < 2; ++x) {
    v.bm[x] = static_cast<uint64_t*>(buffers[MSTF_BUF_BITMAP_K + x]);
    v.val[x] = static_cast<uint16_t*>(buffers[MSTF_BUF_VALUES_K + x]);
    v.off[x] = static_cast<uint32_t*>(buffers[MSTF_BUF_OFFSETS_K + x]);
    v.win[x] = static_cast<uint16_t*>(buffers[MSTF_BUF_WIN_K + x]);
  }
  v.n_comp = static_cast<int32_t*>(buffers[MSTF_BUF_N_COMP]);
  v.n_win = static_cast<int32_t*>(buffers[MSTF_BUF_N_WIN]);
  v.U = c->batch * c->num_kv_heads;
  v.W = c->window;
  v.cap = c->capacity;
  v.keep[0] = c->keep_k;
  v.keep[1] = c->keep_v;
  v.kpad[0] = mstf_k_pad(c->keep_k);
  v.kpad[1] = mstf_k_pad(c->keep_v);
  v.vbits = c->value_bits == 4 ? 4 : 16;
  v.rq[0] = mstf_value_record_bytes(c->keep_k, c->value_bits);
  v.rq[1] = mstf_value_record_bytes(c->keep_v, c->value_bits);
  h->nc.assign(v.U, 0);
  h->nw.assign(v.U, 0);
  *out = h;
  return MSTF_OK;
}

int mstf_cache_destroy(mstf_cache* h) {
  delete h;
  return MSTF_OK;
}

int mstf_cache_counts(const mstf_cache* h, int32_t* n_comp, int32_t* n_win) {
  if (!h) return MSTF_EINVAL;
  if (n_comp) std::memcpy(n_comp, h->nc.data(), sizeof(int32_t) * h->nc.size());
  if (n_win) std::memcpy(n_win, h->nw.data(), sizeof(int32_t) * h->nw.size());
  return MSTF_OK;
}

int mstf_prune_compress_kv(mstf_cache* h, const void* k, const void* v, int32_t T, const int32_t* lengths,
                           void* stream) {
  if (!h) return MSTF_EINVAL;
  if (T < 0) return MSTF_ESHAPE;
  if (T > 0 && (!k || !v || !aligned16(k) || !aligned16(v))) return MSTF_EINVAL;
  const int32_t U = h->view.U, W = h->view.W;
  std::vector<int32_t> nc(U), nw(U);
  for (int32_t u = 0; u < U; ++u) {
    const int32_t L = lengths ? lengths[u] : T;
    if (L < 0 || L > T) return MSTF_EINVAL;
    nw[u] = L < W ? L : W;
    nc[u] = L - nw[u];
    if (nc[u] > h->view.cap) return MSTF_ECAPACITY;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = launch_set_counters(h->view, lengths ? nc.data() : nullptr, lengths ? nw.data() : nullptr, T, s);
  if (e == cudaSuccess)
    e = launch_prefill(h->view, static_cast<const uint16_t*>(k), static_cast<const uint16_t*>(v), T, s);
  if (e != cudaSuccess) return MSTF_ECUDA;
  h->nc = nc;
  h->nw = nw;
  return MSTF_OK;
}

int mstf_append_token(mstf_cache* h, const void* k_new, const void* v_new, void* stream) {
  if (!h || !k_new || !v_new || !aligned16(k_new) || !aligned16(v_new)) return MSTF_EINVAL;
  const int32_t U = h->view.U, W = h->view.W;
  for (int32_t u = 0; u < U; ++u)
    if ((W == 0 || h->nw[u] == W) && h->nc[u] + 1 > h->view.cap) return MSTF_ECAPACITY;
  if (launch_append(h->view, static_cast<const uint16_t*>(k_new), static_cast<const uint16_t*>(v_new),
                    static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return MSTF_ECUDA;
  for (int32_t u = 0; u < U; ++u) {
    if (W == 0 || h->nw[u] == W)
      h->nc[u] += 1;
    else
      h->nw[u] += 1;
  }
  return MSTF_OK;
}

size_t mstf_workspace_bytes(const mstf_cache* h) {
  if (!h) return 0;
  return warp_ws_bytes(h->view.U, h->cfg.num_q_heads / h->cfg.num_kv_heads, sm_count());
}

namespace {
// Host-mirror summary of the counters as the attention will see them (after == true: after one
// decode-step append): stream-K total cost, whether every unit is equal, whether one is empty.
struct MirrorSummary {
  int64_t total_cost;
  bool uniform, empty;
};
MirrorSummary summarize(const mstf_cache* h, bool after) {
  const int32_t U = h->view.U, W = h->view.W;
  MirrorSummary r{0, true, false};
  for (int32_t u = 0; u < U; ++u) {
    int32_t nc = h->nc[u], nw = h->nw[u];
    if (after) {
      if (W == 0 || nw == W) nc += 1; else nw += 1;
    }
    if (nc + nw == 0) r.empty = true;
    r.total_cost += sk_unit_cost(nc, W);
    if (h->nc[u] != h->nc[0] || h->nw[u] != h->nw[0]) r.uniform = false;
  }
  return r;
}

int launch_attention(const mstf_cache* h, const MirrorSummary& ms, bool fuse, const void* k_new, const void* v_new,
              const void* q, float scale, void* out, int32_t out_dtype, float* part_ml, float* part_o, void* ws,
              void* stream) {
  const int32_t G = h->cfg.num_q_heads / h->cfg.num_kv_heads;
  const WarpPlan plan = plan_warp_attention(h->view.U, G, ms.total_cost, h->view.kpad[0], h->view.kpad[1],
                                            h->view.rq[0], h->view.rq[1], sm_count());
  const cudaError_t e = launch_warp_attention(
      h->view, plan, G, ms.uniform ? 1 : 0, fuse ? 1 : 0, static_cast<const uint16_t*>(q), scale,
      static_cast<const uint16_t*>(k_new), static_cast<const uint16_t*>(v_new), out, out_dtype == MSTF_OUT_F16,
      part_ml, part_o, ws, sm_count(), static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? MSTF_OK : MSTF_ECUDA;
}

int check_attention_args(const mstf_cache* h, const void* q, const void* out, int32_t out_dtype, const void* ws,
                         size_t ws_bytes) {
  if (!h || !q || !out || !aligned16(q)) return MSTF_EINVAL;
  if (out_dtype != MSTF_OUT_F32 && out_dtype != MSTF_OUT_F16) return MSTF_EINVAL;
  if (!out_aligned(out, out_dtype)) return MSTF_EINVAL;
  if (!ws || !aligned16(ws) || ws_bytes < mstf_workspace_bytes(h)) return MSTF_EWORKSPACE;
  return MSTF_OK;
}

}  // namespace

int mstf_sparse_decode_attention(const mstf_cache* h, const void* q, float scale, void* out, int32_t out_dtype,
                                 void* ws, size_t ws_bytes, void* stream) {
  const int st = check_attention_args(h, q, out, out_dtype, ws, ws_bytes);
  if (st != MSTF_OK) return st;
  const MirrorSummary ms = summarize(h, false);
  if (ms.empty) return MSTF_EEMPTY;
  return launch_attention(h, ms, false, nullptr, nullptr, q, scale, out, out_dtype, nullptr, nullptr, ws, stream);
}

int mstf_sparse_decode_attention_partial(const mstf_cache* h, const void* q, float scale, float* ml, float* o,
                                         void* ws, size_t ws_bytes, void* stream) {
  const int st = check_attention_args(h, q, ml, MSTF_OUT_F32, ws, ws_bytes);
  if (st != MSTF_OK) return st;
  if (!o || !aligned16(o) || (reinterpret_cast<uintptr_t>(ml) & 7u)) return MSTF_EINVAL;
  const int32_t G = h->cfg.num_q_heads / h->cfg.num_kv_heads;
  bool all_empty = true;
  for (int32_t u = 0; u < h->view.U; ++u) all_empty = all_empty && h->nc[u] + h->nw[u] == 0;
  if (all_empty)  // a shard that holds no token of the sequence (e.g. T < world): the merge identity
    return launch_empty_partials(ml, o, h->view.U * G, static_cast<cudaStream_t>(stream)) == cudaSuccess
               ? MSTF_OK : MSTF_ECUDA;
  const MirrorSummary ms = summarize(h, false);
  if (ms.empty) return MSTF_EEMPTY;
  return launch_attention(h, ms, false, nullptr, nullptr, q, scale, nullptr, MSTF_OUT_F32, ml, o, ws, stream);
}

int mstf_merge_partials(int32_t n, int32_t units, int32_t group, int32_t head_dim, const float* ml, const float* o,
                        void* out, int32_t out_dtype, void* stream) {
  if (n < 1 || units < 0 || group < 1 || !ml || !o || !out) return MSTF_EINVAL;
  if (out_dtype != MSTF_OUT_F32 && out_dtype != MSTF_OUT_F16) return MSTF_EINVAL;
  if (!aligned16(o) || !aligned16(out) || (reinterpret_cast<uintptr_t>(ml) & 7u)) return MSTF_EINVAL;
  if (head_dim != kD || group > kMaxGroup) return MSTF_ENOTSUP;
  return launch_merge_partials(n, units, group, ml, o, out, out_dtype == MSTF_OUT_F16,
                               static_cast<cudaStream_t>(stream)) == cudaSuccess ? MSTF_OK : MSTF_ECUDA;
}

int mstf_decode_step(mstf_cache* h, const void* k_new, const void* v_new, const void* q, float scale, void* out,
                     int32_t out_dtype, void* ws, size_t ws_bytes, void* stream) {
  if (!h || !k_new || !v_new || !aligned16(k_new) || !aligned16(v_new)) return MSTF_EINVAL;
  const int st = check_attention_args(h, q, out, out_dtype, ws, ws_bytes);
  if (st != MSTF_OK) return st;
  const int32_t U = h->view.U, W = h->view.W;
  for (int32_t u = 0; u < U; ++u)
    if ((W == 0 || h->nw[u] == W) && h->nc[u] + 1 > h->view.cap) return MSTF_ECAPACITY;
  const MirrorSummary ms = summarize(h, true);  // counters after the append (a4)
  if (ms.empty) return MSTF_EEMPTY;
  if (!ms.uniform) {  // ragged cache: the two calls in sequence
    const int sa = mstf_append_token(h, k_new, v_new, stream);
    if (sa != MSTF_OK) return sa;
    return mstf_sparse_decode_attention(h, q, scale, out, out_dtype, ws, ws_bytes, stream);
  }
  const int r = launch_attention(h, ms, true, k_new, v_new, q, scale, out, out_dtype, nullptr, nullptr, ws, stream);
  if (r != MSTF_OK) return r;
  for (int32_t u = 0; u < U; ++u) {  // the combine kernel advances the device counters the same way
    if (W == 0 || h->nw[u] == W) h->nc[u] += 1; else h->nw[u] += 1;
  }
  return MSTF_OK;
}

int mstf_decode_step_kernel_count(const mstf_cache* h) {
  if (!h) return MSTF_EINVAL;
  // fused: attention (append inside) + combine; ragged: append + cost prefix + attention + combine
  return summarize(h, true).uniform ? 2 : 4;
}

// Host mirror after `steps` uniform decode steps (unit 0 stands for every unit): window filling
// first, then one compression per step.
static void advance_uniform(int32_t W, int32_t steps, int32_t* nc, int32_t* nw) {
  if (W == 0) { *nc += steps; return; }
  const int32_t fill = std::min(steps, W - *nw);
  *nw += fill;
  *nc += steps - fill;
}

int mstf_graph_step_check(const mstf_cache* h, int32_t steps) {
  if (!h || steps < 0) return MSTF_EINVAL;
  if (!summarize(h, false).uniform) return MSTF_EINVAL;
  int32_t nc = h->nc[0], nw = h->nw[0];
  advance_uniform(h->view.W, steps, &nc, &nw);
  return nc <= h->view.cap ? MSTF_OK : MSTF_ECAPACITY;
}

int mstf_graph_step_commit(mstf_cache* h, int32_t steps) {
  const int st = mstf_graph_step_check(h, steps);
  if (st != MSTF_OK) return st;
  for (int32_t u = 0; u < h->view.U; ++u) advance_uniform(h->view.W, steps, &h->nc[u], &h->nw[u]);
  return MSTF_OK;
}

static int32_t dense_splits(int32_t units, int32_t t_max) {
  const int32_t blocks = (t_max + 15) / 16;
  int32_t s = (3 * 148 + units - 1) / units;
  const int32_t cap_s = blocks / 8 > 1 ? blocks / 8 : 1;
  if (s > cap_s) s = cap_s;
  return s < 1 ? 1 : s;
}

size_t mstf_dense_workspace_bytes(int32_t units, int32_t group, int32_t head_dim, int32_t t_max) {
  if (units < 1 || group < 1 || head_dim != kD || t_max < 1) return 0;
  return dense_ws_bytes(units, group, dense_splits(units, t_max));
}

int mstf_dense_decode_attention(const void* k, const void* v, const int32_t* lengths, int32_t units, int32_t group,
                                int32_t head_dim, int32_t t_max, const void* q, float scale, void* out,
                                int32_t out_dtype, void* ws, size_t ws_bytes, void* stream) {
  if (!k || !v || !lengths || !q || !out || units < 1 || group < 1 || t_max < 1) return MSTF_EINVAL;
  if (head_dim % 64 != 0) return MSTF_ESHAPE;
  if (head_dim != kD || group > kMaxGroup) return MSTF_ENOTSUP;
  if (out_dtype != MSTF_OUT_F32 && out_dtype != MSTF_OUT_F16) return MSTF_EINVAL;
  // uint4 loads of k / v / q rows, float4 partials in the workspace, vector stores of out
  if (!aligned16(k) || !aligned16(v) || !aligned16(q) || !out_aligned(out, out_dtype) ||
      (reinterpret_cast<uintptr_t>(lengths) & 3u))
    return MSTF_EINVAL;
  if (!ws || !aligned16(ws) || ws_bytes < mstf_dense_workspace_bytes(units, group, head_dim, t_max))
    return MSTF_EWORKSPACE;
  if (launch_dense_attention(static_cast<const uint16_t*>(k), static_cast<const uint16_t*>(v), lengths, units,
                             group, t_max, dense_splits(units, t_max), static_cast<const uint16_t*>(q), scale, out,
                             out_dtype == MSTF_OUT_F16, ws, static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return MSTF_ECUDA;
  return MSTF_OK;
}

int mstf_seq_split(int32_t T, int32_t window, int32_t world, int32_t rank, int32_t* t0, int32_t* t1) {
  if (T < 0 || window < 0 || world < 1 || rank < 0 || rank >= world || !t0 || !t1) return MSTF_EINVAL;
  const int64_t C = T - (T < window ? T : window);  // prompt tokens that will be compressed
  *t0 = (int32_t)(C * rank / world);
  *t1 = rank == world - 1 ? T : (int32_t)(C * (rank + 1) / world);
  return MSTF_OK;
}

int mstf_set_key_weights(mstf_cache* h, const float* w) {
  if (!h) return MSTF_EINVAL;
  if (w && !aligned16(w)) return MSTF_EINVAL;
  h->view.kw = w;
  return MSTF_OK;
}

int mstf_query_abs_sum(const void* q, int32_t units, int32_t slots, int32_t group, int32_t head_dim, float* w,
                       void* stream) {
  if (units < 0 || slots < 0 || group < 1 || head_dim < 1) return MSTF_EINVAL;
  if ((long long)units * head_dim > 0 && (!w || (slots > 0 && !q))) return MSTF_EINVAL;
  const cudaError_t e = launch_query_abs_sum(static_cast<const uint16_t*>(q), units, slots, group, head_dim, w,
                                             static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? MSTF_OK : MSTF_ECUDA;
}

int mstf_shard_units(int32_t units, int32_t world, int32_t rank, int32_t* u0, int32_t* u1) {
  if (units < 0 || world < 1 || rank < 0 || rank >= world || !u0 || !u1) return MSTF_EINVAL;
  *u0 = (int32_t)((int64_t)units * rank / world);
  *u1 = (int32_t)((int64_t)units * (rank + 1) / world);
  return MSTF_OK;
}

const char* mstf_status_string(int32_t s) {
  switch (s) {
    case MSTF_OK: return "ok";
    case MSTF_EINVAL: return "invalid argument";
    case MSTF_ESHAPE: return "bad shape (head_dim % 64, heads ratio, or T)";
    case MSTF_EKEEP: return "keep count outside [1, head_dim]";
    case MSTF_ECAPACITY: return "compressed capacity exceeded";
    case MSTF_EEMPTY: return "attention over an empty cache";
    case MSTF_ECUDA: return "CUDA error";
    case MSTF_ENOTSUP: return "unsupported configuration (kernels: head_dim 128, group <= 8)";
    case MSTF_EWORKSPACE: return "workspace missing or too small";
    default: return "unknown status";
  }
}

int mstf_attention_kernel_count(const mstf_cache* h) {
  if (!h) return MSTF_EINVAL;
  return summarize(h, false).uniform ? 2 : 3;  // (+ cost prefix) + attention + combine
}

// Dev tooling (declared in include/mustafar.h, "Development only").
int mstf_dev_read_bandwidth(const void* src, size_t bytes, void* sink, void* stream) {
  if (!src || !sink || !aligned16(src) || (reinterpret_cast<uintptr_t>(sink) & 3u)) return MSTF_EINVAL;
  return launch_dev_read(src, bytes, static_cast<uint32_t*>(sink), sm_count(), static_cast<cudaStream_t>(stream)) ==
                 cudaSuccess ? MSTF_OK : MSTF_ECUDA;
}

int mstf_dev_trace(void* buf) {
  const cudaError_t e = set_dev_trace(buf);
  return e == cudaSuccess ? MSTF_OK : e == cudaErrorNotSupported ? MSTF_ENOTSUP : MSTF_ECUDA;
}

const char* mstf_build_info(void) { return "mustafar-b200 sm_100a (warp-per-worker stream-K, cp.async.bulk + mbarrier, mma.sync m16n8k16, movmatrix)"; }

}  // extern "C"
