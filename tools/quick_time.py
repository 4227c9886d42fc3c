"""Quick device timing of the sparse attention kernel (dev tool, not the bench)."""
import math, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2505_22913_b200 import build as B
B.build()
from paper_2505_22913_b200 import mustafar as M

def run(Bt, hq, hkv, T, keep, layers=8, reps=20):
    U, G = Bt * hkv, hq // hkv
    caches = []
    for l in range(layers):
        K = synth.fp16_torch((U, T, 128), 100 + l); V = synth.fp16_torch((U, T, 128), 200 + l)
        c = M.MustafarCache(Bt, hq, hkv, 128, keep, keep, 32, T)
        c.prune_compress_kv(K, V); del K, V
        caches.append(c)
    q = synth.fp16_torch((U, G, 128), 7)
    out = torch.empty(U, G, 128, device="cuda")
    for c in caches: c.sparse_decode_attention(q, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for r in range(reps):
        for c in caches: c.sparse_decode_attention(q, out=out)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * layers)
    kp = (keep + 7) // 8 * 8
    nbytes = U * (T - 32) * 2 * (16 + 2 * kp) + U * 32 * 512
    dense = U * T * 512
    print(f"B={Bt} hq={hq} hkv={hkv} T={T} keep={keep}: {us:.1f} us/layer  {nbytes/us/1e3:.0f} GB/s compressed  (dense-equiv {dense/us/1e3:.0f} GB/s)", flush=True)
    # dense baseline
    K = synth.fp16_torch((U, T, 128), 1); V = synth.fp16_torch((U, T, 128), 2)
    L = torch.full((U,), T, dtype=torch.int32, device="cuda")
    da = M.DenseAttention(U, G, 128, T)
    da(K, V, L, q, out=out); torch.cuda.synchronize()
    e0.record()
    for r in range(reps): da(K, V, L, q, out=out)
    e1.record(); torch.cuda.synchronize()
    usd = e0.elapsed_time(e1) * 1e3 / reps
    print(f"   own dense: {usd:.1f} us  {dense/usd/1e3:.0f} GB/s (L2-resident if < 126MB: {dense/1e6:.0f} MB)", flush=True)

run(16, 32, 8, 4096, 39)
run(16, 32, 8, 4096, 64)
run(1, 32, 32, 32768, 39)
run(8, 32, 8, 131072, 39, layers=2, reps=5)
