"""Per-CTA / per-segment timeline of one attention launch (dev tool, GPU; sets MSTF_TRACE).
Record per CTA: start, end, smid, nseg, then (segment body end, after combine) pairs."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2505_22913_b200 import mustafar as M
TW = 24

def trace(Bt=16, T=4096, keep=39, hkv=8, hq=32):
    U, G = Bt * hkv, hq // hkv
    K = synth.fp16_torch((U, T, 128), 100); V = synth.fp16_torch((U, T, 128), 200)
    c = M.MustafarCache(Bt, hq, hkv, 128, keep, keep, 32, T); c.prune_compress_kv(K, V); del K, V
    q = synth.fp16_torch((U, G, 128), 7); out = torch.empty(U, G, 128, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    c.sparse_decode_attention(q, out=out)
    flush.fill_(1); torch.cuda.synchronize()
    c.sparse_decode_attention(q, out=out); torch.cuda.synchronize()
    n = TW * 4096
    buf = (ctypes.c_uint64 * n)()
    assert M.lib().mstf_dev_trace(buf, n) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, TW).astype(np.int64)
    a = a[a[:, 0] > 0]
    t0 = a[:, 0].min()
    st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
    nseg = a[:, 3]
    print(f"{os.environ.get('TAG','')} CTAs {len(a)} span {en.max():.1f} us; end p0/p50/max {en.min():.1f}/{np.median(en):.1f}/{en.max():.1f}; "
          f"segments per CTA {np.bincount(nseg).tolist()}", flush=True)
    # per-segment: body duration and combine duration
    body, comb = [], []
    for r in a:
        prev = r[0]
        for i in range(int(r[3])):
            te, tc = r[4 + 2 * i], r[5 + 2 * i]
            body.append((te - prev) / 1e3); comb.append((tc - te) / 1e3); prev = tc
    body, comb = np.array(body), np.array(comb)
    print(f"   segment body p50/p90/max {np.median(body):.1f}/{np.percentile(body,90):.1f}/{body.max():.1f} us; "
          f"combine+ticket p50/p90/max {np.median(comb):.2f}/{np.percentile(comb,90):.2f}/{comb.max():.2f} us", flush=True)
    # first 3 CTAs in detail
    for r in a[:3]:
        segs = [((r[4 + 2 * i] - t0) / 1e3, (r[5 + 2 * i] - t0) / 1e3) for i in range(int(r[3]))]
        print("   cta", [(round(x, 1), round(y, 1)) for x, y in segs], flush=True)

os.environ["MSTF_TRACE"] = "1"
trace()
