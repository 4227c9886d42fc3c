"""Per-layer decode-step time, fused (decode_step) vs append + attention (dev tool, GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2505_22913_b200 import mustafar as M

def run(fused, keep=39, layers=8, reps=10, Bt=16, hq=32, hkv=8, T=4096):
    U, G = Bt * hkv, hq // hkv
    steps = reps + 2
    caches = []
    for l in range(layers):
        K = synth.fp16_torch((U, T, 128), 100 + l); V = synth.fp16_torch((U, T, 128), 200 + l)
        c = M.MustafarCache(Bt, hq, hkv, 128, keep, keep, 32, T + steps); c.prune_compress_kv(K, V); del K, V
        caches.append(c)
    q = synth.fp16_torch((U, G, 128), 7); kn = synth.fp16_torch((U, 128), 8); vn = synth.fp16_torch((U, 128), 9)
    out = torch.empty(U, G, 128, device="cuda")
    def step():
        for c in caches:
            if fused:
                c.decode_step(kn, vn, q, out=out)
            else:
                c.append_token(kn, vn); c.sparse_decode_attention(q, out=out)
    step(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record()
    for r in range(reps): step()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * layers)
if __name__ == "__main__":
    print(os.environ.get("TAG", ""), "unfused %.1f us  fused %.1f us" % (run(False), run(True)), flush=True)
