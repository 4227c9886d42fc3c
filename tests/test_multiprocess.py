"""N>1 path on CPU: torch.distributed gloo, world_size 2.

Units (batch x kv-head pairs) are independent, so a rank owns the contiguous unit range
mstf_shard_units(U, world, rank) (C-ABI host call) and its q / out slices are contiguous in
[B][Hq][d]. Each rank computes its shard (here with the CPU oracle, the per-shard compute of
T4); the gathered result must equal the unsharded computation bit for bit, and the timing
reduction bench.py uses (max over ranks) must pick the slowest rank.
"""
import math
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, U, T, G, q_path, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    from oracle import mustafar_oracle as O
    from paper_2505_22913_b200 import mustafar as M
    d, W, kk = 128, 32, 39
    u0, u1 = M.shard_units(U, world, rank)
    K = synth.fp16_np((U, T, d), 101).view(np.uint16)[u0:u1]
    V = synth.fp16_np((U, T, d), 102).view(np.uint16)[u0:u1]
    q = synth.fp16_np((U, G, d), 103).view(np.uint16)[u0:u1]
    oc = O.OracleCache(u1 - u0, d, kk, kk, W, T)
    oc.prefill(K, V)
    part = torch.from_numpy(O.attention(oc, q, 1 / math.sqrt(d)))          # [U/world, G, d]
    # equal shards here (U % world == 0): all_gather into [U, G, d]
    chunks = [torch.empty_like(part) for _ in range(world)]
    dist.all_gather(chunks, part)
    # bench.py timing rule: the step time is the max over ranks
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        full = torch.cat(chunks).numpy()
        np.save(out_path, full)
        assert t.item() == float(world)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_equals_unsharded(tmp_path, world):
    from paper_2505_22913_b200 import build as B
    B.build()
    import synth
    from oracle import mustafar_oracle as O
    U, T, G, d = 4, 90, 4, 128
    out_path = str(tmp_path / "gathered.npy")
    mp.spawn(_worker, args=(world, _free_port(), U, T, G, None, out_path), nprocs=world, join=True)
    got = np.load(out_path)
    K = synth.fp16_np((U, T, d), 101).view(np.uint16)
    V = synth.fp16_np((U, T, d), 102).view(np.uint16)
    q = synth.fp16_np((U, G, d), 103).view(np.uint16)
    oc = O.OracleCache(U, d, 39, 39, 32, T)
    oc.prefill(K, V)
    ref = O.attention(oc, q, 1 / math.sqrt(d))
    assert np.array_equal(got, ref)


def test_shard_ranges_cover_units_exactly():
    from paper_2505_22913_b200 import build as B
    B.build()
    from paper_2505_22913_b200 import mustafar as M
    for U in (1, 7, 128, 512):
        for world in (1, 2, 3, 4, 8):
            got = [M.shard_units(U, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == U
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [b - a for a, b in got]
            assert max(sizes) - min(sizes) <= 1


def _gather_worker(rank, world, port, U, G, L, out_path):
    """Exactly bench.py's a10 data path: every layer's output tensor is a slice
    full[l][rank*U_r:(rank+1)*U_r] of the [B_global][Hq][d] buffer, written in place by the
    rank's step, then dist.all_gather_into_tensor(full[l], slice) fills the other ranks' rows."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = 128
    Ur = U // world
    full = [torch.empty(world * Ur, G, d, dtype=torch.float16) for _ in range(L)]
    outs = [f[rank * Ur:(rank + 1) * Ur] for f in full]
    for l in range(L):
        # the rank's "step" writes its output slice in place (what decode_step(out=outs[l]) does)
        outs[l].copy_(torch.arange(Ur * G * d, dtype=torch.float32).view(Ur, G, d) * 0.001 + rank + 10 * l)
        assert outs[l].data_ptr() == full[l].data_ptr() + rank * Ur * G * d * 2  # a view, not a copy
        dist.all_gather_into_tensor(full[l], outs[l])
    if rank == 0:
        np.save(out_path, torch.stack(full).float().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_inplace_output_gather_slicing(tmp_path, world):
    """The in-place NCCL all-gather bench.py runs by default for N > 1, with
    gloo on CPU: after the gather every rank's [B][Hq][d] buffer holds each rank's slice in
    rank order (contiguous unit ranges, mstf_shard_units), for every layer."""
    U, G, L = 8, 4, 3
    out_path = str(tmp_path / "full.npy")
    mp.spawn(_gather_worker, args=(world, _free_port(), U, G, L, out_path), nprocs=world, join=True)
    got = np.load(out_path)
    Ur, d = U // world, 128
    base = (np.arange(Ur * G * d, dtype=np.float32).reshape(Ur, G, d) * 0.001)
    for l in range(L):
        for r in range(world):
            exp = (torch.from_numpy(base) + r + 10 * l).half().float().numpy()
            assert np.array_equal(got[l, r * Ur:(r + 1) * Ur], exp), (l, r)
