"""Stream-K grid scan of the fused decode step (dev tool, GPU): for each batch size, the per-layer
step time at several CTA counts (MSTF_SKGRID, read by the planner on every call), 32 layer
caches (> L2). Usage: python tools/grid_scan.py [T] [keep]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2505_22913_b200 import build as B
B.build()
from paper_2505_22913_b200 import mustafar as M


def scan(Bt, T=4096, keep=39, layers=32, reps=6, grids=(16, 32, 48, 64, 96, 148, 222, 296)):
    U, G = Bt * 8, 4
    steps = (reps + 2) * (len(grids) + 1)
    caches = []
    for l in range(layers):
        K = synth.fp16_torch((U, T, 128), 100 + l); V = synth.fp16_torch((U, T, 128), 200 + l)
        c = M.MustafarCache(Bt, 32, 8, 128, keep, keep, 32, T + steps); c.prune_compress_kv(K, V); del K, V
        caches.append(c)
    q = synth.fp16_torch((U, G, 128), 7); kn = synth.fp16_torch((U, 128), 8); vn = synth.fp16_torch((U, 128), 9)
    out = torch.empty(U, G, 128, device="cuda")
    res = []
    for g in (None,) + tuple(grids):
        if g is None:
            os.environ.pop("MSTF_SKGRID", None)
        else:
            os.environ["MSTF_SKGRID"] = str(g)
        for c in caches: c.decode_step(kn, vn, q, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record()
        for r in range(reps):
            for c in caches: c.decode_step(kn, vn, q, out=out)
        e1.record(); torch.cuda.synchronize()
        res.append((g or "default", round(e0.elapsed_time(e1) * 1e3 / (reps * layers), 2)))
    os.environ.pop("MSTF_SKGRID", None)
    print(f"B={Bt} T={T} keep={keep}:", " ".join(f"{g}:{t}" for g, t in res), flush=True)


if __name__ == "__main__":
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    keep = int(sys.argv[2]) if len(sys.argv) > 2 else 39
    for b in (1, 2, 4, 8, 16):
        scan(b, T, keep)
