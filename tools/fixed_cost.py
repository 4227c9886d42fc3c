"""Fixed per-call cost of the attention path: stream launches vs CUDA-graph replay (dev tool, GPU)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2505_22913_b200 import mustafar as M

def run(Bt, T, keep=39, layers=6, reps=20, hkv=8, hq=32):
    U, G = Bt * hkv, hq // hkv
    caches = []
    for l in range(layers):
        K = synth.fp16_torch((U, T, 128), 100 + l); V = synth.fp16_torch((U, T, 128), 200 + l)
        c = M.MustafarCache(Bt, hq, hkv, 128, keep, keep, 32, T); c.prune_compress_kv(K, V); del K, V
        caches.append(c)
    q = synth.fp16_torch((U, G, 128), 7); out = torch.empty(U, G, 128, device="cuda")
    torch.cuda.synchronize()  # prefill ran on the default stream
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for c in caches: c.sparse_decode_attention(q, out=out)
    torch.cuda.synchronize()
    # host cost per call
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for r in range(reps):
            for c in caches: c.sparse_decode_attention(q, out=out)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    host_us = (t1 - t0) * 1e6 / (reps * layers)
    # stream timing
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(s):
        e0.record()
        for r in range(reps):
            for c in caches: c.sparse_decode_attention(q, out=out)
        e1.record()
    torch.cuda.synchronize()
    stream_us = e0.elapsed_time(e1) * 1e3 / (reps * layers)
    # graph replay
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for c in caches: c.sparse_decode_attention(q, out=out)
    g.replay(); torch.cuda.synchronize()
    with torch.cuda.stream(s):
        e0.record()
        for r in range(reps): g.replay()
        e1.record()
    torch.cuda.synchronize()
    graph_us = e0.elapsed_time(e1) * 1e3 / (reps * layers)
    print(f"{os.environ.get('TAG','')} U={U} T={T}: host {host_us:.1f} us/call, stream {stream_us:.1f} us, graph {graph_us:.1f} us", flush=True)

for T in (64, 256, 1024, 4096):
    run(16, T)
