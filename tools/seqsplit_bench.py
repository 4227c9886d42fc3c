"""Sequence-split decode step across GPUs: batch-1 long context.

Each rank holds the token range mstf_seq_split(T, W, world, rank) of every unit (the last rank
also holds the dense window and takes the appends). Per layer and step:
  last rank: mstf_append_token;  every rank: mstf_sparse_decode_attention_partial(q);
  NCCL all_gather of the partials (ml [U][G][2], o [U][G][d] float32) -- the step's one exchange;
  every rank: mstf_merge_partials -> O.
Run: python tools/seqsplit_bench.py [--T 131072 --batch 1 --layers 4]            (1 GPU)
     python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
            tools/seqsplit_bench.py ...                                          (N GPUs)
Prints one JSON line (rank 0): device-timed us per layer-step (max over ranks), tokens/s.
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import synth


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=131072)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--sparsity", type=float, default=0.7)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2505_22913_b200 import build as B
    if rank == 0:
        B.build()
    if world > 1:
        dist.barrier()
    from paper_2505_22913_b200 import mustafar as M

    W, d = 32, 128
    U, G = a.batch * a.hkv, a.hq // a.hkv
    keep = M.keep_from_sparsity(a.sparsity, d)
    T0 = a.T - 1
    nsteps = a.warmup + a.steps
    t0, t1 = M.seq_split(T0, W, world, rank)
    last = rank == world - 1
    caches = []
    for layer in range(a.layers):
        n = t1 - t0
        K = synth.fp16_torch((U, n, d), synth.seed_for(5, 2 * layer) + 7 * rank, device=dev)
        V = synth.fp16_torch((U, n, d), synth.seed_for(5, 2 * layer + 1) + 7 * rank, device=dev)
        c = M.MustafarCache(a.batch, a.hq, a.hkv, d, keep, keep, W if last else 0, n + nsteps + 8, device=dev)
        c.prune_compress_kv(K, V)
        del K, V
        caches.append(c)
    gen = synth.fp16_torch((nsteps, a.layers, U * G * d + 2 * U * d), synth.seed_for(5, 999), device=dev)
    ml = torch.empty(U, G, 2, dtype=torch.float32, device=dev)
    o = torch.empty(U, G, d, dtype=torch.float32, device=dev)
    ml_all = torch.empty(world, U, G, 2, dtype=torch.float32, device=dev)
    o_all = torch.empty(world, U, G, d, dtype=torch.float32, device=dev)
    out = torch.empty(U, G, d, dtype=torch.float16, device=dev)
    scale = 1 / math.sqrt(d)

    def step(s):
        for layer in range(a.layers):
            x = gen[s, layer]
            q = x[:U * G * d].view(U, G, d)
            if last:
                caches[layer].append_token(x[U * G * d:U * G * d + U * d].view(U, d), x[U * G * d + U * d:].view(U, d))
            caches[layer].sparse_decode_attention_partial(q, scale, ml=ml if world > 1 else ml_all[0],
                                                          o=o if world > 1 else o_all[0])
            if world > 1:
                dist.all_gather_into_tensor(ml_all, ml)
                dist.all_gather_into_tensor(o_all, o)
            M.merge_partials(ml_all, o_all, out=out)

    for s in range(a.warmup):
        step(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(a.steps):
        step(a.warmup + s)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / a.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = ms.item()
    assert torch.isfinite(out.float()).all()
    if rank == 0:
        print(json.dumps({
            "tool": "seqsplit_bench", "workload": f"batch {a.batch}, {a.hq}q/{a.hkv}kv, d=128, context {a.T}, "
                                                   f"s={a.sparsity}, {a.layers} layers",
            "n_gpus": world, "scaling": "strong", "steps": a.steps, "warmup": a.warmup,
            "us_per_layer_step": round(ms * 1e3 / a.layers, 3),
            "tokens_per_s": round(a.batch / (ms * 1e-3) * a.layers / 32, 2),
            "tokens_per_s_note": "attention-only decode tokens/s for a 32-layer model (B / (32 x t_layer_step))",
            "rank0_tokens": t1 - t0, "gather_bytes_per_rank_per_layer": U * G * (d + 2) * 4,
        }), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
