"""Sequence split across ranks, CPU side: the oracle's shard partials and
their merge (pinned to the full-cache Algorithm 1, itself pinned to SDPA), the token-range
plan mstf_seq_split (C-ABI host call), and the N>1 path on torch.distributed gloo, world 2:
each rank holds a token range of every unit (window only on the last rank), computes its
partials, all-gathers them and merges; the result equals the unsplit cache's attention.
"""
import math
import os
import socket

import numpy as np
import pytest

import synth
from oracle import mustafar_oracle as O

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

D, KK, W = 128, 39, 32


@pytest.fixture(scope="module")
def M():
    from paper_2505_22913_b200 import build as B
    B.build()
    from paper_2505_22913_b200 import mustafar
    return mustafar


def shard_caches(M, K, V, world, T, kk=KK, window=W):
    """Oracle caches of the split: rank r ingests its prompt range; only the last keeps a window."""
    U = K.shape[0]
    out = []
    for r in range(world):
        t0, t1 = M.seq_split(T, window, world, r)
        w = window if r == world - 1 else 0
        oc = O.OracleCache(U, D, kk, kk, w, max(t1 - t0, 1))
        oc.prefill(K[:, t0:t1], V[:, t0:t1])
        out.append(oc)
    return out


@pytest.mark.parametrize("T", [1, 31, 32, 33, 300])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_seq_split_plan(M, T, world):
    ranges = [M.seq_split(T, W, world, r) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == T
    for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
        assert a1 == b0 and a0 <= a1
    C = T - min(T, W)
    sizes = [b - a for a, b in ranges[:-1]] + [ranges[-1][1] - ranges[-1][0] - min(T, W)]
    assert max(sizes) - min(sizes) <= 1 and sum(sizes) == C      # balanced compressed part
    assert ranges[-1][1] - ranges[-1][0] >= min(T, W)              # last rank holds the window


def test_seq_split_rejects_bad_args(M):
    with pytest.raises(M.MustafarError):
        M.seq_split(10, 32, 2, 2)
    with pytest.raises(M.MustafarError):
        M.seq_split(-1, 32, 2, 0)


def test_partial_single_token():
    """One token: m = s, l = 1, o = v (softmax of one score)."""
    K = synth.fp16_np((1, 1, D), 3).view(np.uint16)
    V = synth.fp16_np((1, 1, D), 4).view(np.uint16)
    q = synth.fp16_np((1, 2, D), 5).view(np.uint16)
    oc = O.OracleCache(1, D, D, D, 0, 1)
    oc.prefill(K, V)
    m, l, o = O.attention_partial(oc, q, 0.5)
    s = 0.5 * (O.fp16_to_f64(q[0]) @ O.fp16_to_f64(K[0, 0]))
    assert np.allclose(m[0], s) and np.array_equal(l[0], [1.0, 1.0])
    assert np.array_equal(o[0], np.stack([O.fp16_to_f64(V[0, 0])] * 2))


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_merged_partials_equal_full_attention(M, world):
    U, T, G = 3, 200, 4
    K = synth.fp16_np((U, T, D), 41).view(np.uint16)
    V = synth.fp16_np((U, T, D), 42).view(np.uint16)
    q = synth.fp16_np((U, G, D), 43).view(np.uint16)
    full = O.OracleCache(U, D, KK, KK, W, T)
    full.prefill(K, V)
    ref = O.attention(full, q, 1 / math.sqrt(D))
    parts = [O.attention_partial(oc, q, 1 / math.sqrt(D)) for oc in shard_caches(M, K, V, world, T)]
    got = O.merge_partials(parts)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_empty_shard_is_identity():
    U, T, G = 2, 50, 2
    K = synth.fp16_np((U, T, D), 51).view(np.uint16)
    V = synth.fp16_np((U, T, D), 52).view(np.uint16)
    q = synth.fp16_np((U, G, D), 53).view(np.uint16)
    oc = O.OracleCache(U, D, KK, KK, W, T)
    oc.prefill(K, V)
    p = O.attention_partial(oc, q, 0.1)
    empty = (np.full((U, G), -np.inf), np.zeros((U, G)), np.zeros((U, G, D)))
    assert np.array_equal(O.merge_partials([p, empty]), O.merge_partials([p]))
    assert np.allclose(O.merge_partials([p]), O.attention(oc, q, 0.1), rtol=0, atol=1e-13)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, U, T, G, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_22913_b200 import mustafar as Mm
    t0, t1 = Mm.seq_split(T, W, world, rank)
    K = synth.fp16_np((U, T, D), 61).view(np.uint16)[:, t0:t1]
    V = synth.fp16_np((U, T, D), 62).view(np.uint16)[:, t0:t1]
    q = synth.fp16_np((U, G, D), 63).view(np.uint16)            # every rank holds the full q
    oc = O.OracleCache(U, D, KK, KK, W if rank == world - 1 else 0, max(t1 - t0, 1))
    oc.prefill(K, V)
    m, l, o = O.attention_partial(oc, q, 1 / math.sqrt(D))
    part = torch.from_numpy(np.concatenate([m[..., None], l[..., None], o], axis=-1))  # [U, G, 2 + d]
    gathered = [torch.empty_like(part) for _ in range(world)]
    dist.all_gather(gathered, part)                           # the one collective of the step
    if rank == 0:
        parts = [(g[..., 0].numpy(), g[..., 1].numpy(), g[..., 2:].numpy()) for g in gathered]
        np.save(out_path, O.merge_partials(parts))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sequence_split(tmp_path, M):
    U, T, G, world = 2, 150, 4, 2
    out_path = str(tmp_path / "merged.npy")
    mp.spawn(_worker, args=(world, _free_port(), U, T, G, out_path), nprocs=world, join=True)
    got = np.load(out_path)
    K = synth.fp16_np((U, T, D), 61).view(np.uint16)
    V = synth.fp16_np((U, T, D), 62).view(np.uint16)
    q = synth.fp16_np((U, G, D), 63).view(np.uint16)
    full = O.OracleCache(U, D, KK, KK, W, T)
    full.prefill(K, V)
    ref = O.attention(full, q, 1 / math.sqrt(D))
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
