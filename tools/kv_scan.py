"""C2_s50 (k_pad 64, TMA kernel) attention time vs env overrides (dev tool, GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2505_22913_b200 import mustafar as M
def run(keep=64, layers=8, reps=10, Bt=16, hq=32, hkv=8, T=4096):
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
    return e0.elapsed_time(e1) * 1e3 / (reps * layers)
if __name__ == "__main__":
    print(os.environ.get("TAG", ""), "keep64 %.1f us" % run(), flush=True)
