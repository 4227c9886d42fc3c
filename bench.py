#!/usr/bin/env python
"""bench.py -- decode-step benchmark of the B200 Mustafar hot path.

A "step" is one decode step of a 32-layer Llama-shaped model's attention over the whole
batch: for every layer, mstf_append_token (prune + compress the token leaving the dense
window) followed by mstf_sparse_decode_attention (Algorithm 1), all
through the C ABI. Synthetic fp16 K/V/Q (seeded counter-based generator, synth/), random
values of the model's shapes; 32 distinct layer caches (> 3 GB) so the working set is far
larger than the 126 MB L2 every step.

    python bench.py [--gpus N --steps K --warmup W] [--workload C2] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (weak scaling: batch per rank fixed)

Rank 0 prints ONE JSON line (metric/value/unit/... see the repo contract in DESIGN.md).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-attn µs/step & HBM GB/s at 70% sparsity; tokens/sec vs dense KV"
LAYERS = 32
W_WINDOW = 32

# BASELINE.json configs; the bench line runs WORKLOADS[args.workload]
WORKLOADS = {
    "C2": dict(desc="Llama-3-8B shape decode, 32 q / 8 kv heads, d=128, 4K context, batch 16, K/V 70% sparsity",
               batch=16, hq=32, hkv=8, T=4096, sk=0.7, sv=0.7),
    "C2_b1": dict(desc="Llama-3-8B shape decode, 4K context, batch 1, K/V 70% sparsity",
                  batch=1, hq=32, hkv=8, T=4096, sk=0.7, sv=0.7),
    "C2_s50": dict(desc="Llama-3-8B shape decode, 4K context, batch 16, K/V 50% sparsity",
                   batch=16, hq=32, hkv=8, T=4096, sk=0.5, sv=0.5),
    "C3": dict(desc="Llama-2-7B shape MHA decode, 32 heads, d=128, 32K context, batch 1, 70% sparsity",
               batch=1, hq=32, hkv=32, T=32768, sk=0.7, sv=0.7),
    "C4": dict(desc="Llama-3-8B shape, 128K context, batch 8, 70% sparsity", batch=8, hq=32, hkv=8, T=131072,
               sk=0.7, sv=0.7),
    "C5": dict(desc="Llama-3-8B shape, 16K context, batch 64 per GPU, 70% sparsity", batch=64, hq=32, hkv=8,
               T=16384, sk=0.7, sv=0.7),
    # NEXT-4: the C4 shape with the prune-then-quantize payload (4-bit codes + fp16 scale / zero per
    # token, tab:joint_quant)
    "C4_q4": dict(desc="Llama-3-8B shape, 128K context, batch 8, 70% sparsity, 4-bit payload (NEXT-4)", batch=8,
                  hq=32, hkv=8, T=131072, sk=0.7, sv=0.7, vbits=4),
    "C2_q4": dict(desc="Llama-3-8B shape decode, 4K context, batch 16, 70% sparsity, 4-bit payload (NEXT-4)",
                  batch=16, hq=32, hkv=8, T=4096, sk=0.7, sv=0.7, vbits=4),
}
DEFAULT_WORKLOAD = "C4"   # the largest single-GPU configuration of BASELINE.json (128K context)
SPEC_HBM_GBS = 8000.0     # nominal B200 HBM3e (DGX figure; B200_PROFILING.md: 7.7 HGX / 8 DGX)


def unit_string(L):
    return f"tokens/s (attention-only decode, {L} layers)"


def config_of(args, cfg, world, L, extra=None):
    """The config object both arms print (the reference arm copies ours)."""
    B = cfg["batch"]
    c = {"workload": args.workload, "desc": cfg["desc"], "batch_per_gpu": B, "global_batch": B * world,
         "num_q_heads": cfg["hq"], "num_kv_heads": cfg["hkv"], "head_dim": 128, "context": cfg["T"],
         "keep_k": keep_of(cfg["sk"]), "keep_v": keep_of(cfg["sv"]), "window": W_WINDOW, "layers": L,
         "value_bits": cfg.get("vbits", 16)}
    if extra:
        c.update(extra)
    return c


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def keep_of(s, d=128):
    return d - math.floor(s * d)


def kpad_of(k):
    return (k + 7) // 8 * 8


def record_bytes(k, vbits=16):
    """Bytes of one token's value record: 2 k_pad (fp16) or the 4-bit record (R26)."""
    return 2 * kpad_of(k) if vbits == 16 else (4 + (k + 1) // 2 + 15) // 16 * 16


def algorithmic_bytes(U, G, n_comp, n_win, keep_k, keep_v, d=128, out_bytes=2, append=False, vbits=16):
    """Bytes one sparse attention call must move: compressed K and V records
    (bitmaps d/8 B + packed values 2*kpad B each; offsets are not read), the dense window,
    q and the output. Split partials are an implementation artefact and are not counted.
    append=True adds one decode step's append (a4): the new K and V tokens read, the evicted
    window tokens read and written back compressed (record + u32 offsets), the new tokens
    written into the ring."""
    rec = (d // 8 + record_bytes(keep_k, vbits)) + (d // 8 + record_bytes(keep_v, vbits))
    b = U * (n_comp * rec + n_win * 4 * d + G * d * 2 + G * d * out_bytes)
    if append:
        b += U * (2 * 2 * d + 2 * 2 * d + rec + 2 * 8 + 2 * 2 * d)
    return b


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region: NVML
    (pynvml) from a background thread every 2 ms, plus one synchronous sample at start() and at
    stop() so even a short region has samples. Falls back to `nvidia-smi -lms 200`."""
    NAMES = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
             ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, dev_index):
        self.dev = dev_index
        self.nv = None
        self.sm, self.reasons, self.mx = [], set(), None
        self.thread = None
        self.stop_flag = False
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[dev_index]) if vis and vis.split(",")[0].isdigit() else dev_index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.nv = pynvml
        except Exception:
            self.nv = None

    def _sample(self):
        nv = self.nv
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        for name, const in self.NAMES:
            if hasattr(nv, const) and r & getattr(nv, const):
                self.reasons.add(name)

    def _loop(self):
        while not self.stop_flag:
            try:
                self._sample()
            except Exception:
                return
            time.sleep(0.002)

    def start(self):
        if self.nv is None:
            self.smi = _SmiSampler(self.dev)
            self.smi.start()
            return
        import threading
        self._sample()
        self.stop_flag = False
        self.thread = threading.Thread(target=self._loop, daemon=True)
        self.thread.start()

    def stop(self):
        if self.nv is None:
            return self.smi.stop()
        self.stop_flag = True
        self.thread.join(timeout=2)
        self._sample()
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml"}


class _SmiSampler:
    """Fallback: nvidia-smi clocks / throttle reasons sampled every 200 ms."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index):
        self.dev = dev_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.dev)], stdout=open(self.path, "w"),
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi"}


# ----------------------------------------------------------------------------- oracle (CPU)
def oracle_sample(cfg, seconds=10.0, max_units=64):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload: per sampled
    unit of layer 0, one decode-step append + Alg. 1 attention in float64. Returns
    (tokens/s extrapolated to the whole workload, description, threads)."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    import synth
    from oracle import mustafar_oracle as O
    B, hq, hkv, T = cfg["batch"], cfg["hq"], cfg["hkv"], cfg["T"]
    U, G, d = B * hkv, hq // hkv, 128
    kk, kv = keep_of(cfg["sk"]), keep_of(cfg["sv"])
    layers = LAYERS
    per_unit = []
    with threadpool_limits(limits=1):
        t_budget = time.perf_counter() + seconds
        for u in range(min(U, max_units)):
            K = synth.fp16_np_rows((U, T, d), synth.seed_for(2, 0), u * T, T).view(np.uint16)
            V = synth.fp16_np_rows((U, T, d), synth.seed_for(2, 1), u * T, T).view(np.uint16)
            oc = O.OracleCache(1, d, kk, kv, W_WINDOW, T + 1, value_bits=cfg.get("vbits", 16))
            oc.prefill(K[None, :T - 1], V[None, :T - 1])
            q = synth.fp16_np_rows((U, G, d), synth.seed_for(2, 2), u * G, G).view(np.uint16)
            t0 = time.perf_counter()
            oc.append(K[None, T - 1], V[None, T - 1])
            O.attention(oc, q[None], 1 / math.sqrt(d))
            per_unit.append(time.perf_counter() - t0)
            if time.perf_counter() > t_budget:
                break
    t_unit = statistics.mean(per_unit)
    step_s = t_unit * U * layers
    desc = (f"{len(per_unit)} units of layer 0 (append + fp64 Alg.1 over {T} tokens each), "
            f"{t_unit * 1e3:.1f} ms/unit, extrapolated x{U} units x{layers} layers; "
            f"host CPU: {cpu_model()}, {os.cpu_count()} logical cores, 1 thread used")
    return B / step_s, desc, 1, t_unit, len(per_unit)


# ----------------------------------------------------------------------------- dense baselines
def dense_baselines(M, B, hq, hkv, d, Tn, t_alloc, scale, dense_k, dense_v, q0, dev, reps=3):
    """Dense-KV decode attention over the same shapes (fp16 KV of `len(dense_k)` layers, rotated
    so the working set exceeds L2): the repo's own dense kernel, torch SDPA, FlashAttention-2
    decode (flash_attn_with_kvcache, split-KV: auto and explicit num_splits) and FlashInfer's
    batch decode on a paged cache (page 16 and 64, CUDA-core and tensor-core variants, planned
    outside the timing). Returns {name: us per layer} and the fastest."""
    import torch
    U, G = B * hkv, hq // hkv
    L = len(dense_k)
    res, notes = {}, {}

    def time_fn(fn):
        for l in range(L):
            fn(l)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            for l in range(L):
                fn(l)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e3 / (reps * L)

    lengths = torch.full((U,), Tn, dtype=torch.int32, device=dev)
    o16 = torch.empty(U, G, d, dtype=torch.float16, device=dev)
    try:
        da = M.DenseAttention(U, G, d, t_alloc, device=dev)
        res["own_dense_kernel"] = time_fn(lambda l: da(dense_k[l], dense_v[l], lengths, q0, scale, out=o16))
    except Exception as ex:  # noqa: BLE001
        notes["own_dense_kernel"] = str(ex)[:120]
    import torch.nn.functional as F
    qs = q0.view(B, hq, 1, d)
    k4 = [k.view(B, hkv, t_alloc, d)[:, :, :Tn] for k in dense_k]
    v4 = [v.view(B, hkv, t_alloc, d)[:, :, :Tn] for v in dense_v]
    try:
        res["torch_sdpa"] = time_fn(lambda l: F.scaled_dot_product_attention(qs, k4[l], v4[l], scale=scale,
                                                                              enable_gqa=True))
    except Exception as ex:  # noqa: BLE001
        notes["torch_sdpa"] = str(ex)[:120]
    # FlashAttention-2 decode: [B, T, Hkv, d] cache (a layout copy, made outside the timing)
    try:
        from flash_attn import flash_attn_with_kvcache
        kf = [x.transpose(1, 2).contiguous() for x in k4]
        vf = [x.transpose(1, 2).contiguous() for x in v4]
        qf = q0.view(B, 1, hq, d)
        best = None
        for ns in (0, 1, 2, 4, 8, 16, 32):
            us = time_fn(lambda l: flash_attn_with_kvcache(qf, kf[l], vf[l], softmax_scale=scale, num_splits=ns))
            if best is None or us < best[0]:
                best = (us, ns)
        res["flash_attn_kvcache"] = best[0]
        notes["flash_attn_kvcache"] = f"num_splits={best[1]} (best of 0=auto,1,2,4,8,16,32)"
        del kf, vf
    except Exception as ex:  # noqa: BLE001
        notes["flash_attn_kvcache"] = str(ex)[:160]
    # FlashInfer batch decode on a paged cache [pages, 2, page, Hkv, d] (NHD)
    try:
        import flashinfer
        ws = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        best = None
        for page in (16, 64):
            npg = (Tn + page - 1) // page
            kv = []
            for l in range(L):
                x = torch.zeros(B * npg, 2, page, hkv, d, dtype=torch.float16, device=dev)
                kb = k4[l].transpose(1, 2)  # [B, Tn, Hkv, d]
                vb = v4[l].transpose(1, 2)
                xs = x.view(B, npg, 2, page, hkv, d)
                full = (Tn // page) * page
                xs[:, :Tn // page, 0] = kb[:, :full].reshape(B, Tn // page, page, hkv, d)
                xs[:, :Tn // page, 1] = vb[:, :full].reshape(B, Tn // page, page, hkv, d)
                if Tn % page:
                    xs[:, Tn // page, 0, :Tn % page] = kb[:, full:]
                    xs[:, Tn // page, 1, :Tn % page] = vb[:, full:]
                kv.append(x)
            indptr = torch.arange(0, B + 1, dtype=torch.int32, device=dev) * npg
            idx = torch.arange(B * npg, dtype=torch.int32, device=dev)
            last = torch.full((B,), Tn - (npg - 1) * page, dtype=torch.int32, device=dev)
            for tc in (False, True):
                w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD", use_tensor_cores=tc)
                w.plan(indptr, idx, last, hq, hkv, d, page, q_data_type=torch.float16, kv_data_type=torch.float16,
                       sm_scale=scale)
                q2 = q0.view(B, hq, d)
                us = time_fn(lambda l: w.run(q2, kv[l]))
                if best is None or us < best[0]:
                    best = (us, page, tc)
            del kv
        res["flashinfer_batch_decode"] = best[0]
        notes["flashinfer_batch_decode"] = f"page_size={best[1]} use_tensor_cores={best[2]} (best of 16/64 x CUDA/tensor cores)"
    except Exception as ex:  # noqa: BLE001
        notes["flashinfer_batch_decode"] = str(ex)[:160]
    return res, notes


# ----------------------------------------------------------------------------- our arm
def run_ours(args, cfg, rank, world, local_rank):
    import numpy as np  # noqa: F401
    import torch
    import torch.distributed as dist

    import synth
    from paper_2505_22913_b200 import build as Bld
    if rank == 0:
        Bld.build()
    if world > 1:
        dist.barrier()
    from paper_2505_22913_b200 import mustafar as M

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    B, hq, hkv, T = cfg["batch"], cfg["hq"], cfg["hkv"], cfg["T"]
    U, G, d = B * hkv, hq // hkv, 128
    kk, kv = keep_of(cfg["sk"]), keep_of(cfg["sv"])
    vbits = cfg.get("vbits", 16)
    L = LAYERS if args.layers is None else args.layers
    K_steps, W_steps = args.steps, args.warmup
    # warm-up, the headline timed pass (no events between a step's kernels, so programmatic
    # dependent launch overlaps them), a second pass with events around every layer call (the
    # roofline's per-launch time), and the end-to-end pass
    total_steps = W_steps + 2 * K_steps + 8 + 2
    T0 = T - 1                       # prefill length; the first decode token makes it T
    cap = T0 - W_WINDOW + total_steps + 8
    scale = 1 / math.sqrt(d)
    gather = args.gather if args.gather is not None else world > 1

    # ---- L layer caches, each prefilled from synthetic K/V; dense copies of a few layers for the
    # dense baselines (enough layers that their working set exceeds the 126 MB L2)
    dense_layers = 0
    if args.dense:
        per_layer_dense = U * (T + total_steps) * d * 2 * 2
        dense_layers = max(2, min(L, -(-3 * 128 * 2**20 // per_layer_dense)))
    caches, dense_k, dense_v, pf_events = [], [], [], []
    for l in range(L):
        seed = synth.seed_for(2, 10 * l + 1000 * rank)
        Kl = synth.fp16_torch((U, T + total_steps, d), seed, device=dev)
        Vl = synth.fp16_torch((U, T + total_steps, d), seed + 1, device=dev)
        c = M.MustafarCache(B, hq, hkv, d, kk, kv, W_WINDOW, cap, device=dev, value_bits=vbits)
        Kp, Vp = Kl[:, :T0].contiguous(), Vl[:, :T0].contiguous()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c.prune_compress_kv(Kp, Vp)   # a1-a4 bulk: one launch of prefill_kernel (+ counters)
        e1.record()
        pf_events.append((e0, e1))
        del Kp, Vp
        caches.append(c)
        if l < dense_layers:
            dense_k.append(Kl)
            dense_v.append(Vl)
        else:
            del Kl, Vl
    torch.cuda.synchronize()
    pf_us = sorted(a.elapsed_time(b) * 1e3 for a, b in pf_events[1:] or pf_events)
    pf_us = pf_us[len(pf_us) // 2]
    kpk, kpv = kpad_of(kk), kpad_of(kv)
    nc0, nw0 = max(T0 - W_WINDOW, 0), min(T0, W_WINDOW)
    pf_bytes = U * (2 * T0 * d * 2 + nc0 * (2 * (d // 8 + 4 * (d // 64)) + record_bytes(kk, vbits) +
                                             record_bytes(kv, vbits)) + 2 * nw0 * d * 2)
    # per-step decode inputs: q [U,G,d], k_new/v_new [U,d] for every (step, layer), one slab per step
    per_layer = U * G * d + 2 * U * d
    gen = synth.fp16_torch((total_steps, L, per_layer), synth.seed_for(2, 7 + rank), device=dev)

    def views(slab, l):
        x = slab[l]
        q = x[:U * G * d].view(U, G, d)
        kn = x[U * G * d:U * G * d + U * d].view(U, d)
        vn = x[U * G * d + U * d:].view(U, d)
        return q, kn, vn

    # outputs: with the a10 gather (default for N > 1) every layer's output is written
    # straight into this rank's slice of the [B_global][Hq][d] tensor and all-gathered in place
    full = [torch.empty(world * U, G, d, dtype=torch.float16, device=dev) for _ in range(L)] if gather else None
    outs = [f[rank * U:(rank + 1) * U] for f in full] if gather else \
        [torch.empty(U, G, d, dtype=torch.float16, device=dev) for _ in range(L)]
    torch.cuda.synchronize()

    # per-(slab, layer) input views built once, outside the timed region: at small batch the
    # step is short enough for per-call Python slicing to starve the GPU
    view_cache = {}
    cur_stream = torch.cuda.current_stream()

    def step(slab, ev=None, do_gather=gather):
        # one decode step per layer: append (a4) + attention (Alg. 1) in one C-ABI call
        # (mstf_decode_step: the append inside the attention launch + the split combine)
        vs = view_cache[slab.data_ptr()]
        for l in range(L):
            q, kn, vn = vs[l]
            if ev is not None:
                ev[l][0].record()
            caches[l].decode_step(kn, vn, q, scale, out=outs[l], stream=cur_stream)
            if ev is not None:
                ev[l][1].record()
            if do_gather:
                dist.all_gather_into_tensor(full[l], outs[l])  # in place: outs[l] is this rank's slice

    for s_ in range(total_steps):
        view_cache[gen[s_].data_ptr()] = [views(gen[s_], l) for l in range(L)]
    sampler = ClockSampler(local_rank)
    attn_ev = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(L)] for _ in range(K_steps)]
    for s in range(W_steps):
        step(gen[s])
    torch.cuda.synchronize()
    # CUDA graph of the whole step (NEXT-1): L x mstf_decode_step captured once, replayed every
    # step on fixed input buffers (the step's inputs are copied in first, one device copy)
    dgraph, gbuf = None, None
    if args.graph:
        gbuf = torch.empty((L, per_layer), dtype=torch.float16, device=dev)
        view_cache[gbuf.data_ptr()] = [views(gbuf, l) for l in range(L)]
        gq, gk, gv = (list(x) for x in zip(*view_cache[gbuf.data_ptr()]))
        dgraph = M.DecodeGraph(caches, gq, gk, gv, outs, scale)

    def run_step(slab, do_gather=gather):
        """The step as the headline times it: one graph replay (or the eager per-layer calls)."""
        if dgraph is None:
            return step(slab, do_gather=do_gather)
        gbuf.copy_(slab, non_blocking=True)
        dgraph.replay()
        if do_gather:
            for l in range(L):
                dist.all_gather_into_tensor(full[l], outs[l])

    if dgraph is not None:  # graph warm-up (its first replay is the captured step)
        for s in range(2):
            run_step(gen[W_steps - 1])
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # ---- headline: K steps, device-timed; an event at every step boundary gives p10/p50/p90
    sampler.start()
    sev = [torch.cuda.Event(enable_timing=True) for _ in range(K_steps + 1)]
    sev[0].record()
    for s in range(K_steps):
        run_step(gen[W_steps + s])
        sev[s + 1].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = sev[0].elapsed_time(sev[K_steps]) / K_steps
    step_ms = sorted(sev[i].elapsed_time(sev[i + 1]) for i in range(K_steps))
    pct = lambda q_: step_ms[min(len(step_ms) - 1, int(round(q_ * (len(step_ms) - 1))))]
    # second timed pass: same step, CUDA events on the launching stream around each layer's call
    for s in range(K_steps):
        step(gen[W_steps + K_steps + s], attn_ev[s], do_gather=False)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    if world > 1:
        dist.barrier()
    attn_ms = [attn_ev[s][l][0].elapsed_time(attn_ev[s][l][1]) for s in range(K_steps) for l in range(L)]
    attn_us = statistics.mean(attn_ms) * 1e3
    # a10 alone: the L in-place all-gathers of one step, device-timed
    gather_us = None
    if gather:
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        g0.record()
        for _ in range(3):
            for l in range(L):
                dist.all_gather_into_tensor(full[l], outs[l])
        g1.record()
        torch.cuda.synchronize()
        gather_us = g0.elapsed_time(g1) * 1e3 / (3 * L)
    nc, nw = caches[0].counts()
    n_comp, n_win = nc[0], nw[0]

    # ---- end to end through the public API with host buffers (pinned), copies inside the timing.
    # Every step copies its inputs (q, k_new, v_new of all layers) host -> device and reads its
    # result (the last layer's output) back to the host. The copy of step s+1 runs on a copy
    # stream while step s computes (double-buffered device inputs); one sync at the end.
    e2e_steps = max(1, min(K_steps, 8, cap - (n_comp + 1)))
    host_in = torch.empty((e2e_steps, L, per_layer), dtype=torch.float16, pin_memory=True)
    host_in.copy_(gen[W_steps:W_steps + e2e_steps].cpu())  # same inputs as the headline pass
    host_out = torch.empty((e2e_steps, U, G, d), dtype=torch.float16, pin_memory=True)
    dev_in = [torch.empty((L, per_layer), dtype=torch.float16, device=dev) for _ in range(2)]
    for b_ in dev_in:
        view_cache[b_.data_ptr()] = [views(b_, l) for l in range(L)]
    copy_stream = torch.cuda.Stream(device=dev)
    compute = torch.cuda.current_stream()
    ready = [torch.cuda.Event() for _ in range(2)]      # inputs of buffer b are on the device
    consumed = [torch.cuda.Event() for _ in range(2)]   # the step reading buffer b has run
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def h2d(s_, b_):
        with torch.cuda.stream(copy_stream):
            dev_in[b_].copy_(host_in[s_], non_blocking=True)
            ready[b_].record(copy_stream)

    f0.record(compute)
    copy_stream.wait_stream(compute)  # the first copy starts inside the timed region
    h2d(0, 0)
    for s in range(e2e_steps):
        b = s % 2
        if s + 1 < e2e_steps:
            if s >= 1:
                copy_stream.wait_event(consumed[1 - b])  # step s-1 has read that buffer
            h2d(s + 1, 1 - b)
        compute.wait_event(ready[b])
        run_step(dev_in[b])
        consumed[b].record(compute)
        host_out[s].copy_(outs[L - 1], non_blocking=True)
    f1.record(compute)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1) / e2e_steps
    assert torch.isfinite(host_out.float()).all()

    # ---- read-only HBM peak (the denominator a pure streaming read reaches on this GPU)
    read_gbs = None
    try:
        buf = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
        sink = torch.zeros(1, dtype=torch.int32, device=dev)
        for _ in range(2):
            M.dev_read_bandwidth(buf, sink)
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record()
        for _ in range(5):
            M.dev_read_bandwidth(buf, sink)
        r1.record()
        torch.cuda.synchronize()
        read_gbs = buf.numel() * 5 / (r0.elapsed_time(r1) * 1e-3) / 1e9
        del buf
    except Exception:  # noqa: BLE001
        read_gbs = None

    # ---- dense-KV baselines (same shapes): the fastest of several implementations
    dense = {}
    if args.dense and dense_k:
        Tn = n_comp + n_win
        q0 = views(gen[0], 0)[0]
        res_d, notes = dense_baselines(M, B, hq, hkv, d, Tn, T + total_steps, scale, dense_k, dense_v, q0, dev)
        dense = {f"{k_}_us_per_layer": round(v_, 3) for k_, v_ in res_d.items()}
        if notes:
            dense["notes"] = notes
        if res_d:
            best_name = min(res_d, key=res_d.get)
            dense["best"] = best_name
            dense["best_dense_us_per_layer"] = round(res_d[best_name], 3)
            dense["dense_bytes_per_layer"] = U * (Tn * 4 * d + 2 * G * d * 2)
            dense["best_dense_achieved_gbs"] = round(dense["dense_bytes_per_layer"] / (res_d[best_name] * 1e-6) / 1e9, 1)
            dense["dense_tok_s_attention_only"] = round(B / (L * res_d[best_name] * 1e-6), 2)
            dense["layers_rotated"] = len(dense_k)
        del dense_k, dense_v

    # ---- reduce over ranks (max time)
    import torch as _t
    vals = _t.tensor([ms, attn_us, e2e_ms, step_ms[0], step_ms[-1]], dtype=_t.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, attn_us, e2e_ms = vals.tolist()[:3]

    bytes_attn = algorithmic_bytes(U, G, n_comp, n_win, kk, kv, append=True, vbits=vbits)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = bytes_attn / (attn_us * 1e-6) / 1e9
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr.get(args.workload, {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    tok_s = world * B / (ms * 1e-3)
    per_step_in = L * per_layer * 2
    nk = caches[0].decode_step_kernel_count()
    par = f"dp{world} (batch x kv-head units" + (", in-place NCCL all_gather of every layer's output)" if gather
                                                 else ", no collective)")
    res = {
        "metric": METRIC,
        "value": round(tok_s, 2),
        "unit": unit_string(L),
        "n_gpus": world, "steps": K_steps, "warmup": W_steps,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f16 (fp32 accumulate)" if vbits == 16 else "u4 codes + f16 scale/zero (fp16 MMA, fp32 accumulate)",
        "data": "synthetic (seeded splitmix64 -> fp16 ~N(0,1)); no model weights",
        "config": config_of(args, cfg, world, L, {
            "parallelism": par,
            "l2": f"inputs larger than L2: {L} layer caches x {caches[0].nbytes / 1e6:.0f} MB"}),
        "us_per_layer_step": round(ms * 1e3 / L, 3),
        "step_ms_p10_p50_p90": [round(pct(0.1), 4), round(pct(0.5), 4), round(pct(0.9), 4)],
        "decode_step_us_per_call_events": round(attn_us, 3),  # second pass: events around each call
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "frac_of_spec_8tbs": round(achieved / SPEC_HBM_GBS, 4),
                     "read_peak_gbs": round(read_gbs, 1) if read_gbs else None,
                     "frac_of_read_peak": round(achieved / read_gbs, 4) if read_gbs else None,
                     "kernel": ("mstf_decode_step: mstf_attn_warp_kernel (append fused) + mstf_warp_combine_kernel"
                                if nk == 2 else "mstf_decode_step: append + attention + combine")
                               + ", CUDA events around each call in a second timed pass",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if peaks else "fallback 6.65 TB/s",
                     "read_peak_source": "mstf_dev_read_bandwidth over 4 GiB, 5 passes, measured in this run",
                     "algorithmic_bytes_per_launch": bytes_attn},
        "e2e": {"value": round(world * B / (e2e_ms * 1e-3), 2), "unit": unit_string(L),
                "h2d_bytes_per_step": per_step_in, "d2h_bytes_per_step": U * G * d * 2,
                "steps": e2e_steps, "ms_per_step": round(e2e_ms, 4)},
        "gpu_launches": K_steps * L * nk,  # headline pass (graph replays launch the same kernels)
        "step_launch": "one CUDA graph replay per step (L x mstf_decode_step captured)" if dgraph is not None
                       else "eager: L mstf_decode_step calls per step",
        "clocks": clocks,
        "dense_kv": dense,
        "prefill": {"kernel": "prefill_kernel (mstf_prune_compress_kv: a1-a4 bulk over the prompt)",
                    "tokens": T0, "us_per_layer": round(pf_us, 2),
                    "achieved_gbs": round(pf_bytes / (pf_us * 1e-6) / 1e9, 1), "peak": peak,
                    "frac": round(pf_bytes / (pf_us * 1e-6) / 1e9 / peak, 4), "algorithmic_bytes": pf_bytes,
                    "timing": "CUDA events around each layer's call during setup, median over layers 1.."},
    }
    if gather_us is not None:
        res["multi_gpu"] = {"kernel_only_us_per_layer": round(attn_us, 3), "gather_us_per_layer": round(gather_us, 3),
                            "e2e_ms_per_step": round(e2e_ms, 4), "collective": "NCCL all_gather_into_tensor, in place"}
    if dense.get("best_dense_us_per_layer"):
        # our whole step (append + attention, headline pass) vs dense attention alone
        res["speedup_vs_best_dense_attention"] = round(dense["best_dense_us_per_layer"] / (ms * 1e3 / L), 3)
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        v, desc, cores, _, _ = oracle_sample(cfg, seconds=args.cpu_seconds)
        res["cpu_baseline"] = {"value": round(v, 4), "unit": unit_string(L), "cores": cores, "kind": "oracle",
                               "sample": desc}
    return res


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU oracle as it stands, on the host cores (rank 0 only). Each step
    is a bounded sample of the workload: one unit of layer 0 (a decode-step append + fp64
    Algorithm 1 over its tokens); ms_per_step is that measured sample time, and `value`
    extrapolates it to the whole job (units x layers), on our arm's metric, unit and config."""
    if rank != 0:
        return None
    per_unit, desc = [], ""
    for s in range(args.warmup + args.steps):
        v, desc, cores, t_unit, _ = oracle_sample(cfg, seconds=0.0, max_units=1)
        if s >= args.warmup:
            per_unit.append(t_unit)
    t_unit = statistics.mean(per_unit)
    B, U = cfg["batch"], cfg["batch"] * cfg["hkv"]
    v = B / (t_unit * U * LAYERS)
    return {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": unit_string(LAYERS),
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_unit * 1e3, 3),
            "ms_per_step_note": "measured time of one step's bounded sample (1 unit of 1 layer); value = "
                                f"global_batch / (that x {U} units x {LAYERS} layers)",
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded splitmix64 -> fp16 ~N(0,1)); no model weights",
            "config": config_of(args, cfg, world, LAYERS, {"parallelism": "CPU oracle, 1 thread"}),
            "cpu_baseline": {"value": round(v, 6), "unit": unit_string(LAYERS), "cores": cores, "kind": "oracle",
                             "sample": "each step: " + desc},
            "e2e": {"value": round(v, 6), "unit": unit_string(LAYERS), "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=list(WORKLOADS))
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--no-dense", dest="dense", action="store_false")
    ap.add_argument("--gather", dest="gather", action="store_true", default=None,
                    help="all-gather every layer's output into [B][Hq][d] (a10; default on for N > 1)")
    ap.add_argument("--no-gather", dest="gather", action="store_false")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch the 32 layer calls eagerly instead of replaying one CUDA graph per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference", "at least 3 warm-up steps"
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    cfg = WORKLOADS[args.workload]
    if args.impl == "reference":
        res = run_reference(args, cfg, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res = run_ours(args, cfg, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
