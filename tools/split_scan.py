"""Scan split counts for the sparse attention on a few configs (dev tool)."""
import os, sys, math, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2505_22913_b200 import mustafar as M
cfgs = [(16, 32, 8, 4096, 39, 8), (16, 32, 8, 4096, 64, 8), (1, 32, 32, 32768, 39, 8), (8, 32, 8, 131072, 39, 2)]
for (Bt, hq, hkv, T, keep, layers) in cfgs:
    U, G = Bt * hkv, hq // hkv
    caches = []
    for l in range(layers):
        K = synth.fp16_torch((U, T, 128), 100 + l); V = synth.fp16_torch((U, T, 128), 200 + l)
        c = M.MustafarCache(Bt, hq, hkv, 128, keep, keep, 32, T); c.prune_compress_kv(K, V); del K, V
        caches.append(c)
    q = synth.fp16_torch((U, G, 128), 7); out = torch.empty(U, G, 128, device="cuda")
    kp = (keep + 7) // 8 * 8
    nbytes = U * (T - 32) * 2 * (16 + 2 * kp) + U * 32 * 512
    res = []
    for S in [0, 1, 2, 3, 4, 6, 8, 9, 12, 16, 24, 37]:
        if S: os.environ["MSTF_SPLITS"] = str(S)
        else: os.environ.pop("MSTF_SPLITS", None)
        for c in caches: c.sparse_decode_attention(q, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for r in range(10):
            for c in caches: c.sparse_decode_attention(q, out=out)
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (10 * layers)
        res.append(f"S={S}:{us:.1f}")
    print(f"B={Bt} hkv={hkv} T={T} keep={keep}: " + " ".join(res), flush=True)
    del caches
