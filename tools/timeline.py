"""Kernel timeline of a few decode layer-steps via torch.profiler/CUPTI (dev tool, GPU):
per-kernel durations and the idle gaps between consecutive kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from torch.profiler import profile, ProfilerActivity
from paper_2505_22913_b200 import mustafar as M

Bt, hq, hkv, T, keep, L = 16, 32, 8, 4096, 39, 8
U, G = Bt * hkv, hq // hkv
caches = []
for l in range(L):
    K = synth.fp16_torch((U, T, 128), 100 + l); V = synth.fp16_torch((U, T, 128), 200 + l)
    c = M.MustafarCache(Bt, hq, hkv, 128, keep, keep, 32, T + 64); c.prune_compress_kv(K, V); del K, V
    caches.append(c)
q = synth.fp16_torch((U, G, 128), 7); kn = synth.fp16_torch((U, 128), 8); vn = synth.fp16_torch((U, 128), 9)
out = torch.empty(U, G, 128, device="cuda", dtype=torch.float16)
APPEND = os.environ.get("APPEND", "1") == "1"
def step():
    for c in caches:
        if APPEND:
            c.append_token(kn, vn)
        c.sparse_decode_attention(q, out=out)
step(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
prev_end = None
rows = []
for e in ev:
    s, t = e.time_range.start, e.time_range.end
    gap = (s - prev_end) if prev_end is not None else 0
    rows.append((e.name[:60], t - s, gap))
    prev_end = t
import collections
agg = collections.defaultdict(list)
for n, d, g in rows[len(rows) // 3:]:
    agg[n].append((d, g))
print(os.environ.get("TAG", ""))
for n, v in agg.items():
    ds = sorted(x[0] for x in v); gs = sorted(x[1] for x in v)
    print(f"{n:60s} n={len(v):3d} dur med {ds[len(ds)//2]:.1f} us  gap-before med {gs[len(gs)//2]:.1f} us")
