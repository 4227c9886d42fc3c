"""Batch / sparsity / context sweep of the decode step against the dense-KV baselines (dev tool).

Runs bench.run_ours (the bench's own timed step, CUDA events, L2-busting layer rotation) for
the Llama-3-8B attention shape over BASELINE.json's C2 batch range (1..16) at 50% and 70%
sparsity, and longer contexts at batch 1, and prints one line per point:
  workload, us per layer-step (append + attention), best dense us (fastest of own kernel, torch
  SDPA, FlashAttention-2 decode, FlashInfer batch decode),
  sparse/dense speed ratio, roofline frac.
Usage: python tools/batch_sweep.py [--layers 32]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)  # >= 126 MB L2 of sparse data even at B=1
    ap.add_argument("--steps", type=int, default=6)
    a = ap.parse_args()
    pts = [(b, 4096, s) for s in (0.7, 0.5) for b in (1, 2, 4, 8, 16)]
    pts += [(1, 16384, 0.7), (1, 65536, 0.7), (4, 32768, 0.7)]
    for b, T, s in pts:
        cfg = dict(desc=f"Llama-3-8B shape, B={b}, T={T}, s={s}", batch=b, hq=32, hkv=8, T=T, sk=s, sv=s,
                   layers=a.layers)
        args = argparse.Namespace(steps=a.steps, warmup=3, layers=a.layers, dense=True, gather=False, graph=True,
                                  no_cpu_baseline=True, cpu_seconds=0, workload="sweep")
        r = bench.run_ours(args, cfg, 0, 1, 0)
        d = r["dense_kv"]
        best = d.get("best_dense_us_per_layer")
        step = r["us_per_layer_step"]
        print(json.dumps({"B": b, "T": T, "s": s, "us_per_layer_step": step,
                          "best_dense": d.get("best"), "best_dense_us": best,
                          "dense_over_sparse": round(best / step, 3) if best else None,
                          "roofline_frac": r["roofline"]["frac"]}), flush=True)


if __name__ == "__main__":
    main()
