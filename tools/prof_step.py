"""One decode layer-step (append + attention) a few times, for ncu launch lists (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2505_22913_b200 import mustafar as M
Bt, hq, hkv, T, keep = 16, 32, 8, 4096, 39
U, G = Bt * hkv, hq // hkv
K = synth.fp16_torch((U, T, 128), 100); V = synth.fp16_torch((U, T, 128), 200)
c = M.MustafarCache(Bt, hq, hkv, 128, keep, keep, 32, T + 16)
c.prune_compress_kv(K[:, :T - 8].contiguous(), V[:, :T - 8].contiguous())
q = synth.fp16_torch((U, G, 128), 7); out = torch.empty(U, G, 128, device="cuda", dtype=torch.float16)
for i in range(6):
    c.append_token(K[:, T - 8 + i].contiguous(), V[:, T - 8 + i].contiguous())
    c.sparse_decode_attention(q, out=out)
torch.cuda.synchronize(); print("ok")
