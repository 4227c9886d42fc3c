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
       "merged_us": [round(float(rel[:, 4][w[:, 4] > 0].min()), 2), round(float(rel[:, 4][w[:, 4] > 0].max()), 2)] if bool((w[:, 4] > 0).any()) else None,
       "done_us": [round(float(rel[:, 3][w[:, 3] > 0].min()), 2), round(float(rel[:, 3][w[:, 3] > 0].median()), 2), round(float(rel[:, 3][w[:, 3] > 0].max()), 2)],
       "combine_start_us": [round(float(((comb[:, 0] - t0) / 1e3).min()), 2), round(float(((comb[:, 0] - t0) / 1e3).max()), 2)] if len(comb) else None,
       "combine_done_us": [round(float(((comb[:, 1] - t0) / 1e3).min()), 2), round(float(((comb[:, 1] - t0) / 1e3).max()), 2)] if len(comb) else None}
# appenders (fused step): workers whose append phase took > 0.5 us
ph = rel[:, 1] - rel[:, 0]
app = ph > float(ph.median()) + 1.0
if bool(app.any()):
    res["appenders"] = int(app.sum())
    res["appender_done_us"] = [round(float(rel[app, 3].median()), 2), round(float(rel[app, 3].max()), 2)]
    res["appender_first_block_us"] = [round(float(rel[app, 2].median()), 2), round(float(rel[app, 2].max()), 2)]
    res["other_done_us"] = [round(float(rel[~app, 3].median()), 2), round(float(rel[~app, 3].max()), 2)]
print(json.dumps(res), flush=True)
res = {}
# per-CTA spread (workers = CTA * wpc + warp; wpc from the number of active workers / 148 if full)
wpc = int(sys.argv[4]) if len(sys.argv) > 4 else 16
d = (tr[:65536, 3].double() - t0) / 1e3
act_all = tr[:65536, 0] > 0
nw = int(act_all.sum())
if nw % wpc == 0 and nw // wpc <= 148:
    dd = d[:nw].view(nw // wpc, wpc)
    cta_max = dd.max(1).values
    cta_min = dd.min(1).values
    res["cta_done_max_us"] = [round(float(cta_max.min()), 2), round(float(cta_max.median()), 2), round(float(cta_max.max()), 2)]
    res["within_cta_spread_us_median"] = round(float((cta_max - cta_min).median()), 2)
    res["done_by_warp_idx_mean_us"] = [round(float(x), 1) for x in dd.mean(0)]
    fb = (tr[:nw, 2].double() - t0) / 1e3
    res["first_block_by_warp_idx_mean_us"] = [round(float(x), 2) for x in fb.view(nw // wpc, wpc).mean(0)]
print(json.dumps(res), flush=True)
