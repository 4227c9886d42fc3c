"""Thin Python binding of the C ABI in include/mustafar.h (argument marshalling only).

Every step of the hot path runs in the CUDA kernels of lib/libmustafar.so; this module only
allocates device buffers with torch, passes pointers/sizes/streams through ctypes and maps
status codes to exceptions. There is no CPU fallback: if the library or a CUDA device is
missing, calls raise.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libmustafar.so")

# must match include/mustafar.h
STATUS = {0: "MSTF_OK", -1: "MSTF_EINVAL", -2: "MSTF_ESHAPE", -3: "MSTF_EKEEP", -4: "MSTF_ECAPACITY",
          -5: "MSTF_EEMPTY", -6: "MSTF_ECUDA", -7: "MSTF_ENOTSUP", -8: "MSTF_EWORKSPACE"}
BUFFERS = ("bitmap_k", "bitmap_v", "values_k", "values_v", "offsets_k", "offsets_v",
           "win_k", "win_v", "n_comp", "n_win")
NUM_BUFFERS = len(BUFFERS)
OUT_F32, OUT_F16 = 0, 1
EXPORTS = ("mstf_keep_from_sparsity", "mstf_k_pad", "mstf_value_record_bytes", "mstf_cache_buffer_bytes", "mstf_cache_create",
           "mstf_cache_destroy", "mstf_cache_counts", "mstf_prune_compress_kv", "mstf_append_token",
           "mstf_workspace_bytes", "mstf_sparse_decode_attention", "mstf_dense_workspace_bytes",
           "mstf_dense_decode_attention", "mstf_shard_units", "mstf_decode_step",
           "mstf_decode_step_kernel_count", "mstf_attention_kernel_count",
           "mstf_set_key_weights", "mstf_query_abs_sum",
           "mstf_seq_split", "mstf_sparse_decode_attention_partial", "mstf_merge_partials",
           "mstf_dev_read_bandwidth", "mstf_dev_trace", "mstf_graph_step_check", "mstf_graph_step_commit",
           "mstf_status_string", "mstf_build_info")


class MustafarError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn}: {STATUS.get(status, status)} ({msg})")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("batch", "num_q_heads", "num_kv_heads", "head_dim", "keep_k", "keep_v", "window", "capacity",
                 "value_bits")]


_lib = None


def lib() -> ctypes.CDLL:
    """Load lib/libmustafar.so (build it with paper_2505_22913_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2505_22913_b200.build`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
    sig = {
        "mstf_keep_from_sparsity": (i32, [ctypes.c_double, i32]),
        "mstf_k_pad": (i32, [i32]),
        "mstf_value_record_bytes": (i32, [i32, i32]),
        "mstf_cache_buffer_bytes": (ctypes.c_int, [ctypes.POINTER(Config), ctypes.POINTER(sz)]),
        "mstf_cache_create": (ctypes.c_int, [ctypes.POINTER(Config), ctypes.POINTER(vp), ctypes.POINTER(vp)]),
        "mstf_cache_destroy": (ctypes.c_int, [vp]),
        "mstf_cache_counts": (ctypes.c_int, [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)]),
        "mstf_prune_compress_kv": (ctypes.c_int, [vp, vp, vp, i32, ctypes.POINTER(i32), vp]),
        "mstf_append_token": (ctypes.c_int, [vp, vp, vp, vp]),
        "mstf_workspace_bytes": (sz, [vp]),
        "mstf_sparse_decode_attention": (ctypes.c_int, [vp, vp, ctypes.c_float, vp, i32, vp, sz, vp]),
        "mstf_dense_workspace_bytes": (sz, [i32, i32, i32, i32]),
        "mstf_dense_decode_attention": (ctypes.c_int, [vp, vp, vp, i32, i32, i32, i32, vp, ctypes.c_float,
                                                       vp, i32, vp, sz, vp]),
        "mstf_shard_units": (ctypes.c_int, [i32, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)]),
        "mstf_decode_step": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_float, vp, i32, vp, sz, vp]),
        "mstf_decode_step_kernel_count": (ctypes.c_int, [vp]),
        "mstf_attention_kernel_count": (ctypes.c_int, [vp]),
        "mstf_set_key_weights": (ctypes.c_int, [vp, vp]),
        "mstf_query_abs_sum": (ctypes.c_int, [vp, i32, i32, i32, i32, vp, vp]),
        "mstf_seq_split": (ctypes.c_int, [i32, i32, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)]),
        "mstf_sparse_decode_attention_partial": (ctypes.c_int, [vp, vp, ctypes.c_float, vp, vp, vp, sz, vp]),
        "mstf_merge_partials": (ctypes.c_int, [i32, i32, i32, i32, vp, vp, vp, i32, vp]),
        "mstf_dev_read_bandwidth": (ctypes.c_int, [vp, sz, vp, vp]),
        "mstf_dev_trace": (ctypes.c_int, [vp]),
        "mstf_graph_step_check": (ctypes.c_int, [vp, i32]),
        "mstf_graph_step_commit": (ctypes.c_int, [vp, i32]),
        "mstf_status_string": (ctypes.c_char_p, [i32]),
        "mstf_build_info": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        try:
            f = getattr(L, name)
        except AttributeError:
            if name.startswith("mstf_dev_"):  # development hooks: optional (A/B of older builds)
                continue
            raise
        f.restype, f.argtypes = res, args
    _lib = L
    return L


def _check(fn: str, st: int):
    if st != 0:
        raise MustafarError(fn, st, lib().mstf_status_string(st).decode())


def _stream(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _dev_ptr(t: torch.Tensor, dtype=torch.float16, name="tensor") -> int:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (the hot path has no CPU fallback)")
    if t.dtype != dtype or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous {dtype} tensor")
    return t.data_ptr()


def _expect(t: torch.Tensor, shape, name: str):
    """Shape guard before a pointer crosses the C ABI (the library sees only pointers and
    sizes, so a wrong-sized tensor would be read or written out of bounds on the device)."""
    if tuple(t.shape) != tuple(shape):
        # accept any view with the same element count and contiguous layout ([B, H, d] == [U, G, d])
        if t.numel() != math.prod(shape):
            raise ValueError(f"{name}: expected shape {tuple(shape)} ({math.prod(shape)} elements), "
                             f"got {tuple(t.shape)}")


def keep_from_sparsity(s: float, d: int) -> int:
    return int(lib().mstf_keep_from_sparsity(float(s), int(d)))


def k_pad(keep: int) -> int:
    return int(lib().mstf_k_pad(int(keep)))


def shard_units(units: int, world: int, rank: int):
    a, b = ctypes.c_int32(), ctypes.c_int32()
    _check("mstf_shard_units", lib().mstf_shard_units(units, world, rank, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def query_abs_sum(q: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Output-aware accumulator: q fp16 [U, R, G, d] (R window queries of each unit's
    G query heads) -> float32 [U, d], w = sum_r sum_g |q| (mstf_query_abs_sum)."""
    U, R, G, d = q.shape
    if out is None:
        out = torch.empty(U, d, dtype=torch.float32, device=q.device)
    _expect(out, (U, d), "out")
    _check("mstf_query_abs_sum", lib().mstf_query_abs_sum(_dev_ptr(q, name="q"), U, R, G, d,
                                                          _dev_ptr(out, torch.float32, "out"), _stream(stream)))
    return out


def seq_split(T: int, window: int, world: int, rank: int):
    """Prompt token range [t0, t1) of `rank` in a sequence split (mstf_seq_split)."""
    a, b = ctypes.c_int32(), ctypes.c_int32()
    _check("mstf_seq_split", lib().mstf_seq_split(T, window, world, rank, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def merge_partials(ml: torch.Tensor, o: torch.Tensor, out=None, out_dtype=torch.float32, stream=None):
    """Merge shard partials ml float32 [n, U, G, 2], o float32 [n, U, G, d] -> out [U, G, d]
    (mstf_merge_partials)."""
    n, U, G, d = o.shape
    _expect(ml, (n, U, G, 2), "ml")
    if out is None:
        out = torch.empty(U, G, d, dtype=out_dtype, device=o.device)
    code = OUT_F16 if out.dtype == torch.float16 else OUT_F32
    _check("mstf_merge_partials", lib().mstf_merge_partials(n, U, G, d, _dev_ptr(ml, torch.float32, "ml"),
                                                            _dev_ptr(o, torch.float32, "o"),
                                                            _dev_ptr(out, out.dtype, "out"), code, _stream(stream)))
    return out


def dev_read_bandwidth(x: torch.Tensor, sink: torch.Tensor, stream=None):
    """Development only: stream the bytes of x once (read-only HBM roofline measurement)."""
    if not x.is_cuda or not x.is_contiguous():
        raise ValueError("x must be a contiguous CUDA tensor")
    _check("mstf_dev_read_bandwidth", lib().mstf_dev_read_bandwidth(x.data_ptr(), x.numel() * x.element_size(),
                                                                    _dev_ptr(sink, torch.int32, "sink"),
                                                                    _stream(stream)))


def dev_trace(buf: torch.Tensor | None):
    """Development only: record the attention kernel's per-worker phase stamps into buf (int64
    CUDA tensor, >= (65536 + units) x 8 entries), or stop recording (None)."""
    if buf is not None and (not buf.is_cuda or buf.dtype != torch.int64 or not buf.is_contiguous()):
        raise ValueError("buf must be a contiguous int64 CUDA tensor")
    _check("mstf_dev_trace", lib().mstf_dev_trace(None if buf is None else buf.data_ptr()))


def buffer_bytes(cfg: Config):
    sizes = (ctypes.c_size_t * NUM_BUFFERS)()
    _check("mstf_cache_buffer_bytes", lib().mstf_cache_buffer_bytes(ctypes.byref(cfg), sizes))
    return [int(x) for x in sizes]


@dataclass
class Shape:
    batch: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int = 128

    @property
    def units(self):
        return self.batch * self.num_kv_heads

    @property
    def group(self):
        return self.num_q_heads // self.num_kv_heads


class MustafarCache:
    """One compressed KV cache (one layer, all (batch, kv-head) units) on one device."""

    def __init__(self, batch, num_q_heads, num_kv_heads, head_dim, keep_k, keep_v, window, capacity,
                 device=None, value_bits=16):
        self.cfg = Config(batch, num_q_heads, num_kv_heads, head_dim, keep_k, keep_v, window, capacity, value_bits)
        self.value_bits = value_bits
        self.shape = Shape(batch, num_q_heads, num_kv_heads, head_dim)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        sizes = buffer_bytes(self.cfg)
        # one slab, every buffer 256-byte aligned
        offs, tot = [], 0
        for s in sizes:
            offs.append(tot)
            tot += (s + 255) // 256 * 256
        self._slab = torch.empty(max(tot, 256), dtype=torch.uint8, device=self.device)
        base = self._slab.data_ptr()
        self._raw = {n: self._slab[o:o + s] for n, o, s in zip(BUFFERS, offs, sizes)}
        self._raw["n_comp"].zero_()   # an empty cache (the host mirror starts at 0 too)
        self._raw["n_win"].zero_()
        ptrs = (ctypes.c_void_p * NUM_BUFFERS)(*[base + o for o in offs])
        h = ctypes.c_void_p()
        _check("mstf_cache_create", lib().mstf_cache_create(ctypes.byref(self.cfg), ptrs, ctypes.byref(h)))
        self._h = h
        self._ws = torch.zeros(max(int(lib().mstf_workspace_bytes(self._h)), 256), dtype=torch.uint8,
                               device=self.device)
        self.keep_k, self.keep_v, self.window, self.capacity = keep_k, keep_v, window, capacity

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.mstf_cache_destroy(h)
            self._h = None

    @property
    def units(self):
        return self.shape.units

    @property
    def nbytes(self):
        return self._slab.numel()

    def buffers(self):
        """Typed views of the device buffers (layout of include/mustafar.h)."""
        U, cap, d, W = self.units, self.capacity, self.shape.head_dim, max(self.window, 1)
        nt = d // 64
        r = self._raw
        return {
            "bitmap_k": r["bitmap_k"].view(torch.int64).view(U, cap, nt),
            "bitmap_v": r["bitmap_v"].view(torch.int64).view(U, cap, nt),
            # the values buffers end with a 16-byte tail guard (include/mustafar.h)
            "values_k": self._values_view(r["values_k"], self.keep_k),
            "values_v": self._values_view(r["values_v"], self.keep_v),
            "offsets_k": r["offsets_k"].view(torch.int32).view(U, cap, nt),
            "offsets_v": r["offsets_v"].view(torch.int32).view(U, cap, nt),
            "win_k": r["win_k"].view(torch.int16).view(U, W, d),
            "win_v": r["win_v"].view(torch.int16).view(U, W, d),
            "n_comp": r["n_comp"].view(torch.int32),
            "n_win": r["n_win"].view(torch.int32),
        }

    def _values_view(self, raw, keep):
        U, cap = self.units, self.capacity
        rq = int(lib().mstf_value_record_bytes(int(keep), int(self.value_bits)))
        if self.value_bits == 4:  # 4-bit records [U][cap][rq] bytes
            return raw[:U * cap * rq].view(U, cap, rq)
        return raw[:U * cap * rq].view(torch.int16).view(U, cap, rq // 2)

    def attention_kernel_count(self) -> int:
        """Kernels launched by one sparse_decode_attention call on this cache."""
        n = lib().mstf_attention_kernel_count(self._h)
        if n < 0:
            _check("mstf_attention_kernel_count", n)
        return n

    def counts(self):
        U = self.units
        a, b = (ctypes.c_int32 * U)(), (ctypes.c_int32 * U)()
        _check("mstf_cache_counts", lib().mstf_cache_counts(self._h, a, b))
        return list(a), list(b)

    def prune_compress_kv(self, k: torch.Tensor, v: torch.Tensor, lengths=None, stream=None):
        """k, v: fp16 [U, T, d] (== [B, Hkv, T, d]) on the device."""
        T = k.shape[-2]
        d = self.shape.head_dim
        _expect(k, (self.units, T, d), "k")
        _expect(v, (self.units, T, d), "v")
        ln = None
        if lengths is not None:
            if len(lengths) != self.units:
                raise ValueError(f"lengths: expected {self.units} entries, got {len(lengths)}")
            ln = (ctypes.c_int32 * self.units)(*[int(x) for x in lengths])
        _check("mstf_prune_compress_kv",
               lib().mstf_prune_compress_kv(self._h, _dev_ptr(k, name="k"), _dev_ptr(v, name="v"), T, ln,
                                            _stream(stream)))

    def sparse_decode_attention_partial(self, q: torch.Tensor, scale=None, ml=None, o=None, stream=None):
        """Softmax partials of this cache's tokens (one shard of a sequence split):
        ml float32 [U, G, 2] (m in log2 units, l), o float32 [U, G, d] unnormalised
        (mstf_sparse_decode_attention_partial)."""
        d, U, G = self.shape.head_dim, self.units, self.shape.group
        scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
        _expect(q, (U, G, d), "q")
        if ml is None:
            ml = torch.empty(U, G, 2, dtype=torch.float32, device=self.device)
        if o is None:
            o = torch.empty(U, G, d, dtype=torch.float32, device=self.device)
        _expect(ml, (U, G, 2), "ml")
        _expect(o, (U, G, d), "o")
        _check("mstf_sparse_decode_attention_partial",
               lib().mstf_sparse_decode_attention_partial(self._h, _dev_ptr(q, name="q"), scale,
                                                          _dev_ptr(ml, torch.float32, "ml"),
                                                          _dev_ptr(o, torch.float32, "o"), self._ws.data_ptr(),
                                                          self._ws.numel(), _stream(stream)))
        return ml, o

    def set_key_weights(self, w: torch.Tensor | None):
        """Output-aware K pruning for later K compressions: w float32 [U, d] on the device
        (read by the kernels at run time; keep it alive and update it in stream order), or None
        for magnitude pruning (mstf_set_key_weights)."""
        if w is not None:
            _expect(w, (self.units, self.shape.head_dim), "w")
        ptr = None if w is None else _dev_ptr(w, torch.float32, "w")
        _check("mstf_set_key_weights", lib().mstf_set_key_weights(self._h, ptr))
        self._kw = w

    def append_token(self, k_new: torch.Tensor, v_new: torch.Tensor, stream=None):
        """k_new, v_new: fp16 [U, d] (== [B, Hkv, d]) on the device."""
        _expect(k_new, (self.units, self.shape.head_dim), "k_new")
        _expect(v_new, (self.units, self.shape.head_dim), "v_new")
        _check("mstf_append_token", lib().mstf_append_token(self._h, _dev_ptr(k_new, name="k_new"),
                                                           _dev_ptr(v_new, name="v_new"), _stream(stream)))

    def decode_step(self, k_new: torch.Tensor, v_new: torch.Tensor, q: torch.Tensor, scale=None, out=None,
                    out_dtype=torch.float32, stream=None):
        """append_token(k_new, v_new) then sparse_decode_attention(q) -- one fused launch when the
        cache is uniform (mstf_decode_step). Returns out [U, G, d]."""
        d = self.shape.head_dim
        scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
        _expect(k_new, (self.units, d), "k_new")
        _expect(v_new, (self.units, d), "v_new")
        _expect(q, (self.units, self.shape.group, d), "q")
        if out is None:
            out = torch.empty((self.units, self.shape.group, d), dtype=out_dtype, device=self.device)
        _expect(out, (self.units, self.shape.group, d), "out")
        code = OUT_F16 if out.dtype == torch.float16 else OUT_F32
        _check("mstf_decode_step",
               lib().mstf_decode_step(self._h, _dev_ptr(k_new, name="k_new"), _dev_ptr(v_new, name="v_new"),
                                      _dev_ptr(q, name="q"), scale, _dev_ptr(out, out.dtype, "out"), code,
                                      self._ws.data_ptr(), self._ws.numel(), _stream(stream)))
        return out

    def decode_step_kernel_count(self) -> int:
        """Kernels one decode_step call launches in the cache's current state."""
        n = lib().mstf_decode_step_kernel_count(self._h)
        if n < 0:
            _check("mstf_decode_step_kernel_count", n)
        return n

    def sparse_decode_attention(self, q: torch.Tensor, scale=None, out=None, out_dtype=torch.float32,
                                stream=None):
        """q: fp16 [U, G, d] (== [B, Hq, d]). Returns out [U, G, d] (fp32 or fp16)."""
        d = self.shape.head_dim
        scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
        _expect(q, (self.units, self.shape.group, d), "q")
        if out is None:
            out = torch.empty((self.units, self.shape.group, d), dtype=out_dtype, device=self.device)
        _expect(out, (self.units, self.shape.group, d), "out")
        code = OUT_F16 if out.dtype == torch.float16 else OUT_F32
        _check("mstf_sparse_decode_attention",
               lib().mstf_sparse_decode_attention(self._h, _dev_ptr(q, name="q"), scale,
                                                  _dev_ptr(out, out.dtype, "out"), code, self._ws.data_ptr(),
                                                  self._ws.numel(), _stream(stream)))
        return out


class DenseAttention:
    """Dense-KV decode attention baseline (same kernel skeleton, no pruning)."""

    def __init__(self, units, group, head_dim, t_max, device=None):
        self.units, self.group, self.head_dim, self.t_max = units, group, head_dim, t_max
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        n = int(lib().mstf_dense_workspace_bytes(units, group, head_dim, t_max))
        if n == 0:
            raise MustafarError("mstf_dense_workspace_bytes", -7, "unsupported shape")
        self._ws = torch.empty(n, dtype=torch.uint8, device=self.device)

    def __call__(self, k, v, lengths, q, scale=None, out=None, out_dtype=torch.float32, stream=None):
        scale = 1.0 / math.sqrt(self.head_dim) if scale is None else float(scale)
        U, G, d = self.units, self.group, self.head_dim
        _expect(k, (U, self.t_max, d), "k")
        _expect(v, (U, self.t_max, d), "v")
        _expect(lengths, (U,), "lengths")
        _expect(q, (U, G, d), "q")
        if out is None:
            out = torch.empty((U, G, d), dtype=out_dtype, device=self.device)
        _expect(out, (U, G, d), "out")
        code = OUT_F16 if out.dtype == torch.float16 else OUT_F32
        _check("mstf_dense_decode_attention",
               lib().mstf_dense_decode_attention(_dev_ptr(k, name="k"), _dev_ptr(v, name="v"),
                                                 _dev_ptr(lengths, torch.int32, "lengths"), self.units,
                                                 self.group, self.head_dim, self.t_max, _dev_ptr(q, name="q"),
                                                 scale, _dev_ptr(out, out.dtype, "out"), code,
                                                 self._ws.data_ptr(), self._ws.numel(), _stream(stream)))
        return out


class DecodeGraph:
    """A CUDA graph of one decode step over several layer caches (NEXT-1): for every layer,
    mstf_decode_step(k_new[l], v_new[l], q[l]) -> out[l] -- the fused append + attention launch
    and the split combine, chained with programmatic dependent launch. Capture records the
    launches once; replay() re-runs them with no host work per layer. The kernels read the
    per-unit counters from the device, so step after step the replays see the growing cache;
    the host mirrors are advanced by mstf_graph_step_commit. Inputs and outputs are the fixed
    buffers given here: write the next step's q / k_new / v_new into them before replay()."""

    def __init__(self, caches, q, k_new, v_new, out, scale=None, stream=None):
        self.caches = list(caches)
        n = len(self.caches)
        assert len(q) == len(k_new) == len(v_new) == len(out) == n
        for c in self.caches:
            _check("mstf_graph_step_check", lib().mstf_graph_step_check(c._h, 1))
        self.q, self.k_new, self.v_new, self.out = q, k_new, v_new, out
        self.scale = scale
        self.graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=self.caches[0].device) if stream is None else stream
        self._stream = s
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.graph.capture_begin()
            try:
                for l, c in enumerate(self.caches):
                    c.decode_step(k_new[l], v_new[l], q[l], scale, out=out[l], stream=s)
            finally:
                self.graph.capture_end()
        # capture enqueued nothing on the device, but decode_step advanced the host mirrors by
        # one step: step them back by re-syncing from the pre-capture state is not possible, so
        # the first replay() is the step the capture described (no commit for it)
        self._pending = 1
        torch.cuda.current_stream().wait_stream(s)

    def replay(self):
        """One decode step of every layer (asynchronous on the capture stream's device order:
        the graph is launched on the current stream)."""
        if self._pending == 0:
            for c in self.caches:
                _check("mstf_graph_step_check", lib().mstf_graph_step_check(c._h, 1))
        self.graph.replay()
        if self._pending:
            self._pending -= 1
        else:
            for c in self.caches:
                _check("mstf_graph_step_commit", lib().mstf_graph_step_commit(c._h, 1))
