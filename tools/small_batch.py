"""dev: small-batch latency breakdown (C2_b1 shape by default): per-layer time of the attention
call alone, the fused decode step, and the append alone, each replayed as a CUDA graph of L
layer calls.  python tools/small_batch.py [B] [T] [L]"""
import sys, json, torch
sys.path.insert(0, ".")
from paper_2505_22913_b200 import mustafar as M

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
T = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
L = int(sys.argv[3]) if len(sys.argv) > 3 else 32
Hq, Hkv, d, W = 32, 8, 128, 32
U, G = B * Hkv, Hq // Hkv
torch.manual_seed(0)
dev = torch.device("cuda")
caches = []
for l in range(L):
    c = M.MustafarCache(B, Hq, Hkv, d, 39, 39, W, T + 64, device=dev)
    k = torch.randn(U, T, d, device=dev, dtype=torch.float16)
    v = torch.randn(U, T, d, device=dev, dtype=torch.float16)
    c.prune_compress_kv(k, v)
    caches.append(c)
q = [torch.randn(U, G, d, device=dev, dtype=torch.float16) for _ in range(L)]
kn = [torch.randn(U, d, device=dev, dtype=torch.float16) for _ in range(L)]
vn = [torch.randn(U, d, device=dev, dtype=torch.float16) for _ in range(L)]
out = [torch.empty(U, G, d, device=dev, dtype=torch.float32) for _ in range(L)]
torch.cuda.synchronize()


def graph_time(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn(s)  # warm (uncaptured: sets function attributes)
        g = torch.cuda.CUDAGraph()
        g.capture_begin()
        fn(s)
        g.capture_end()
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps / L


res = {"B": B, "T": T, "L": L}
res["attention_us"] = graph_time(lambda s: [c.sparse_decode_attention(q[i], out=out[i], stream=s) for i, c in enumerate(caches)])
res["attention_kernels"] = caches[0].attention_kernel_count()
# decode steps grow the caches: capacity T + 64 allows the warm-up + capture-free replays below
res["append_us"] = graph_time(lambda s: [c.append_token(kn[i], vn[i], stream=s) for i, c in enumerate(caches)], reps=5)
print(json.dumps(res), flush=True)
