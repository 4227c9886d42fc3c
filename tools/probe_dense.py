"""Probe external dense decode baselines (flashinfer, flash_attn, SDPA) on C2 shapes (dev tool)."""
import math, time, torch, sys
B, hq, hkv, T, d = 16, 32, 8, 4096, 128
dev = "cuda"
L = 16
K = [torch.randn(B, hkv, T, d, dtype=torch.float16, device=dev) for _ in range(L)]
V = [torch.randn(B, hkv, T, d, dtype=torch.float16, device=dev) for _ in range(L)]
q = torch.randn(B, hq, d, dtype=torch.float16, device=dev)
def tm(fn, reps=5):
    for l in range(L): fn(l)
    torch.cuda.synchronize(); a=torch.cuda.Event(True); b=torch.cuda.Event(True); a.record()
    for _ in range(reps):
        for l in range(L): fn(l)
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b)*1e3/(reps*L)
nbytes = B*hkv*T*d*2*2
import torch.nn.functional as F
us = tm(lambda l: F.scaled_dot_product_attention(q.view(B,hq,1,d), K[l], V[l], enable_gqa=True)); print("sdpa", us, nbytes/us/1e3, "GB/s", flush=True)
try:
    from flash_attn import flash_attn_with_kvcache
    kk = [k.transpose(1,2).contiguous() for k in K]; vv = [v.transpose(1,2).contiguous() for v in V]
    us = tm(lambda l: flash_attn_with_kvcache(q.view(B,1,hq,d), kk[l], vv[l])); print("flash_attn", us, nbytes/us/1e3, flush=True)
    del kk, vv
except Exception as e: print("flash_attn fail", repr(e)[:200], flush=True)
try:
    import flashinfer
    t0=time.time()
    ws = torch.empty(256<<20, dtype=torch.uint8, device=dev)
    w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "HND")
    # one page per sequence, page_size = T
    indptr = torch.arange(B+1, dtype=torch.int32, device=dev); idx = torch.arange(B, dtype=torch.int32, device=dev)
    last = torch.full((B,), T, dtype=torch.int32, device=dev)
    w.plan(indptr, idx, last, hq, hkv, d, T, data_type=torch.float16, q_data_type=torch.float16)
    kv = [torch.stack([K[l], V[l]], dim=1) for l in range(L)]  # [B(pages), 2, hkv, T, d]
    us = tm(lambda l: w.run(q, kv[l])); print("flashinfer", us, nbytes/us/1e3, "plan+jit s", time.time()-t0, flush=True)
except Exception as e: print("flashinfer fail", repr(e)[:300], flush=True)
