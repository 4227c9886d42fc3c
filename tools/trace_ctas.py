"""Per-worker timeline of one attention launch (dev tool, GPU; sets MSTF_TRACE): when each
K/V warp pair finishes, relative to the kernel start."""
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
    ke = (a[:, 4:8] - t0).ravel() / 1e3
    ve = (a[:, 8:12] - t0).ravel() / 1e3
    segs = a[:, 12:16].ravel()
    pc = lambda x: "/".join(f"{np.percentile(x, q):.1f}" for q in (0, 10, 50, 90, 100))
    print(f"{os.environ.get('TAG','')} workers {len(ve)}: K end p0/10/50/90/100 {pc(ke)}; V end {pc(ve)} us; "
          f"V-K lag p50 {np.median(ve - ke):.1f}; segments {np.bincount(segs).tolist()}", flush=True)
    # slow workers: by segments
    for s_ in np.unique(segs):
        print(f"   {s_} segments: V end mean {ve[segs == s_].mean():.1f} us (n={int((segs == s_).sum())})")
    np.save("gpurun_out/worker_ends.npy", np.stack([ke, ve, segs]))

os.environ["MSTF_TRACE"] = "1"
trace()
