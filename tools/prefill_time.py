"""Device timing of the bulk prune+compress (prefill) path, mstf_prune_compress_kv (dev tool).

Per call: read 2 tensors x U x T x d fp16, write bitmaps + packed values + offsets for the
compressed tokens and the dense window rows. Reports us/call and algorithmic GB/s.
Usage: python tools/prefill_time.py [B hq hkv T keep]   (default: C2 layer, B=16, 4K, s=.7)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2505_22913_b200 import build as B

B.build()
from paper_2505_22913_b200 import mustafar as M


def algorithmic_bytes(U, T, W, keep, d=128):
    kp = (keep + 7) // 8 * 8
    nc, nw = max(T - W, 0), min(T, W)
    rd = 2 * U * T * d * 2
    wr = 2 * U * (nc * (d // 8 + 2 * kp + 4 * d // 64) + nw * d * 2)
    return rd + wr


def run(Bt=16, hq=32, hkv=8, T=4096, keep=39, reps=10, W=32, vbits=16):
    U = Bt * hkv
    K = synth.fp16_torch((U, T, 128), 11)
    V = synth.fp16_torch((U, T, 128), 12)
    caches = [M.MustafarCache(Bt, hq, hkv, 128, keep, keep, W, T + 8, value_bits=vbits) for _ in range(2)]
    for c in caches:
        c.prune_compress_kv(K, V)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for r in range(reps):
        caches[r & 1].prune_compress_kv(K, V)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    nb = algorithmic_bytes(U, T, W, keep)
    print(f"prefill U={U} T={T} keep={keep} vbits={vbits}: {us:.1f} us/call, {nb / 1e6:.1f} MB, {nb / us / 1e3:.0f} GB/s",
          flush=True)
    return us, nb


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    if a:
        run(*a)
    else:
        run()
        run(keep=64)
        run(Bt=1, hq=32, hkv=32, T=32768, keep=39)
