"""Compare the stream-K and split schedules with each other and the oracle (dev tool, GPU)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from oracle import mustafar_oracle as O
from paper_2505_22913_b200 import mustafar as M

def case(B, hq, hkv, T, keep, W, lengths=None, sample=(0,)):
    U, G, d = B * hkv, hq // hkv, 128
    K = synth.fp16_torch((U, T, d), 11); V = synth.fp16_torch((U, T, d), 12); q = synth.fp16_torch((U, G, d), 13)
    c = M.MustafarCache(B, hq, hkv, d, keep, keep, W, T)
    c.prune_compress_kv(K, V, lengths=lengths) if lengths is not None else c.prune_compress_kv(K, V)
    outs = {}
    for sc in ("split", "sk"):
        os.environ["MSTF_SCHED"] = sc
        outs[sc] = c.sparse_decode_attention(q, 1 / math.sqrt(d)).cpu().numpy().astype(np.float64)
    os.environ.pop("MSTF_SCHED")
    dif = np.abs(outs["split"] - outs["sk"]).max()
    errs = []
    Kh = K.cpu().view(torch.int16).numpy().view(np.uint16); Vh = V.cpu().view(torch.int16).numpy().view(np.uint16)
    qh = q.cpu().view(torch.int16).numpy().view(np.uint16)
    for u in sample:
        n = T if lengths is None else int(lengths[u])
        oc = O.OracleCache(1, d, keep, keep, W, T); oc.prefill(Kh[u:u+1, :n], Vh[u:u+1, :n])
        ref = O.attention(oc, qh[u][None], 1 / math.sqrt(d))[0]
        for sc in ("split", "sk"):
            o = outs[sc][u]
            errs.append((sc, u, float((np.abs(o - ref).max(-1) / np.abs(ref).max(-1)).max())))
    bad = [e for e in errs if not e[2] <= 2e-3]
    print(f"B={B} hkv={hkv} T={T} keep={keep} W={W} ragged={lengths is not None}: split-vs-sk {dif:.2e}", "BAD " + str(bad) if bad else "ok", flush=True)

case(16, 32, 8, 4096, 39, 32, sample=(0, 77, 127))
case(1, 32, 8, 4096, 64, 32, sample=(0, 7))
case(2, 8, 2, 1000, 39, 32, sample=(0, 1, 2, 3))
case(3, 8, 2, 777, 39, 0, lengths=[777, 5, 300, 1, 64, 65], sample=(0, 1, 2, 3, 4, 5))
case(4, 8, 2, 500, 39, 32, lengths=[1, 40, 33, 500, 17, 16, 32, 48], sample=tuple(range(8)))
case(64, 8, 2, 300, 39, 32, lengths=[(37 * i) % 300 + 1 for i in range(128)], sample=(0, 5, 127))
case(1, 4, 1, 20, 39, 32, sample=(0,))
