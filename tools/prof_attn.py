"""Run the sparse attention a few times on one config (for ncu capture; dev tool)."""
import math, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2505_22913_b200 import build as B
B.build()
from paper_2505_22913_b200 import mustafar as M
Bt, hq, hkv, T, keep = [int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (16, 32, 8, 4096, 39))]
U, G = Bt * hkv, hq // hkv
K = synth.fp16_torch((U, T, 128), 100); V = synth.fp16_torch((U, T, 128), 200)
c = M.MustafarCache(Bt, hq, hkv, 128, keep, keep, 32, T)
c.prune_compress_kv(K, V); del K, V
q = synth.fp16_torch((U, G, 128), 7)
out = torch.empty(U, G, 128, device="cuda")
for i in range(5):
    c.sparse_decode_attention(q, out=out)
torch.cuda.synchronize()
print("done")
