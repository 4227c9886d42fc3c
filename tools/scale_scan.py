"""Attention time vs context length and unit count (dev tool, GPU): slope = per-token cost,
intercept = fixed cost (launch, ramp, combine)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2505_22913_b200 import mustafar as M

def run(Bt, T, keep=39, layers=6, reps=10, hkv=8, hq=32):
    U, G = Bt * hkv, hq // hkv
    caches = []
    for l in range(layers):
        K = synth.fp16_torch((U, T, 128), 100 + l); V = synth.fp16_torch((U, T, 128), 200 + l)
        c = M.MustafarCache(Bt, hq, hkv, 128, keep, keep, 32, T); c.prune_compress_kv(K, V); del K, V
        caches.append(c)
    q = synth.fp16_torch((U, G, 128), 7); out = torch.empty(U, G, 128, device="cuda")
    for c in caches: c.sparse_decode_attention(q, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record()
    for r in range(reps):
        for c in caches: c.sparse_decode_attention(q, out=out)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * layers)
    mb = U * T * 2 * (16 + 2 * 40) / 1e6
    print(f"{os.environ.get('TAG','')} B={Bt} U={U} T={T}: {us:.1f} us  {mb:.1f} MB  {mb/us:.2f} TB/s", flush=True)
    del caches

for T in (1024, 2048, 4096, 8192, 16384):
    run(16, T)
for Bt in (4, 8, 32):
    run(Bt, 4096)
