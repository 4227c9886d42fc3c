"""dev: phase timeline of the attention kernel (mstf_dev_trace): per-worker start, after the
fused appends, first block landed, done; combine CTAs start/done.
python tools/trace_attn.py B T [fused]"""
import sys, json, torch
sys.path.insert(0, ".")
from paper_2505_22913_b200 import mustafar as M

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
T = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
fused = len(sys.argv) > 3 and sys.argv[3] == "fused"
Hq, Hkv, d, W = 32, 8, 128, 32
U, G = B * Hkv, Hq // Hkv
dev = torch.device("cuda")
c = M.MustafarCache(B, Hq, Hkv, d, 39, 39, W, T + 64, device=dev)
c.prune_compress_kv(torch.randn(U, T, d, device=dev, dtype=torch.float16), torch.randn(U, T, d, device=dev, dtype=torch.float16))
q = torch.randn(U, G, d, device=dev, dtype=torch.float16)
kn = torch.randn(U, d, device=dev, dtype=torch.float16)
out = torch.empty(U, G, d, device=dev, dtype=torch.float32)
buf = torch.zeros((65536 + U) * 8, dtype=torch.int64, device=dev)
for it in range(3):
    buf.zero_()
    M.dev_trace(buf)
    if fused:
        c.decode_step(kn, kn, q, out=out)
    else:
        c.sparse_decode_attention(q, out=out)
    torch.cuda.synchronize()
    M.dev_trace(None)
tr = buf.view(-1, 8).cpu()
w = tr[:65536]
act = w[:, 0] > 0
w = w[act].double()
t0 = w[:, 0].min()
rel = (w - t0) / 1e3  # us
comb = tr[65536:65536 + U].double()
comb = comb[comb[:, 0] > 0]
res = {"B": B, "T": T, "fused": fused, "workers": int(act.sum()),
       "start_us": [round(float(rel[:, 0].min()), 2), round(float(rel[:, 0].median()), 2), round(float(rel[:, 0].max()), 2)],
       "after_append_us": [round(float(rel[:, 1].median()), 2), round(float(rel[:, 1].max()), 2)],
       "first_block_us": [round(float(rel[:, 2][w[:, 2] > 0].min()), 2), round(float(rel[:, 2][w[:, 2] > 0].median()), 2), round(float(rel[:, 2][w[:, 2] > 0].max()), 2)],
       "done_us": [round(float(rel[:, 3][w[:, 3] > 0].min()), 2), round(float(rel[:, 3][w[:, 3] > 0].median()), 2), round(float(rel[:, 3][w[:, 3] > 0].max()), 2)],
       "combine_start_us": [round(float(((comb[:, 0] - t0) / 1e3).min()), 2), round(float(((comb[:, 0] - t0) / 1e3).max()), 2)] if len(comb) else None,
       "combine_done_us": [round(float(((comb[:, 1] - t0) / 1e3).min()), 2), round(float(((comb[:, 1] - t0) / 1e3).max()), 2)] if len(comb) else None}
print(json.dumps(res), flush=True)
