"""Per-CTA timeline of one attention launch (dev tool, GPU; needs MSTF_TRACE=1)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2505_22913_b200 import mustafar as M

def trace(Bt=16, T=4096, keep=39, hkv=8, hq=32):
    U, G = Bt * hkv, hq // hkv
    K = synth.fp16_torch((U, T, 128), 100); V = synth.fp16_torch((U, T, 128), 200)
    c = M.MustafarCache(Bt, hq, hkv, 128, keep, keep, 32, T); c.prune_compress_kv(K, V); del K, V
    q = synth.fp16_torch((U, G, 128), 7); out = torch.empty(U, G, 128, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    c.sparse_decode_attention(q, out=out)
    flush.fill_(1); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); c.sparse_decode_attention(q, out=out); e1.record(); torch.cuda.synchronize()
    n = 3 * 8192
    buf = (ctypes.c_uint64 * n)()
    assert M.lib().mstf_dev_trace(buf, n) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 3).astype(np.int64)
    a = a[a[:, 0] > 0]
    t0 = a[:, 0].min()
    st, en, sm = a[:, 0] - t0, a[:, 1] - t0, a[:, 2]
    dur = en - st
    print(f"{os.environ.get('TAG','')} T={T} event {e0.elapsed_time(e1)*1e3:.1f} us; CTAs {len(a)}; span {en.max()/1e3:.1f} us; "
          f"start p0/p50/max {np.percentile(st,0)/1e3:.1f}/{np.percentile(st,50)/1e3:.1f}/{st.max()/1e3:.1f} us; "
          f"dur min/p50/max {dur.min()/1e3:.1f}/{np.percentile(dur,50)/1e3:.1f}/{dur.max()/1e3:.1f} us; "
          f"end min/p50/max {en.min()/1e3:.1f}/{np.percentile(en,50)/1e3:.1f}/{en.max()/1e3:.1f} us", flush=True)
    # which CTAs are slow: by SM id group, by CTA index (data location)
    order = np.argsort(sm)
    g = sm // 16
    print("   mean dur by smid//16:", [round(float(dur[g == i].mean()) / 1e3, 1) for i in range(10) if (g == i).any()])
    ci = np.arange(len(a)) * 10 // len(a)
    print("   mean dur by CTA-index decile:", [round(float(dur[ci == i].mean()) / 1e3, 1) for i in range(10)])
    # SM pairs: do both CTAs of an SM run slow together?
    sm_mean = {int(s_): float(dur[sm == s_].mean()) for s_ in np.unique(sm)}
    v = np.array(list(sm_mean.values()))
    print("   per-SM mean dur p0/p50/p100: %.1f/%.1f/%.1f us" % (v.min() / 1e3, np.median(v) / 1e3, v.max() / 1e3))
    within = [float(np.ptp(dur[sm == s_])) for s_ in np.unique(sm) if (sm == s_).sum() == 2]
    print("   within-SM dur spread median %.1f us" % (np.median(within) / 1e3 if within else 0))
    np.save(f"gpurun_out/trace_{os.environ.get('RUN','0')}.npy", np.stack([st, en, sm, np.arange(len(a))]))
    per_sm = np.bincount(sm, minlength=148)
    print("   CTAs per SM histogram:", np.bincount(per_sm).tolist())
    # busy fraction per SM over the span
    hist = np.histogram(en / 1e3, bins=10, range=(0, en.max() / 1e3))[0]
    print("   CTA end-time histogram (10 bins over span):", hist.tolist())

os.environ["MSTF_TRACE"] = "1"
for r in range(3):
    os.environ['RUN'] = str(r)
    trace(T=4096)
