"""CUDA-graph replay of the decode step (NEXT-1): one graph of L layers x mstf_decode_step,
replayed step after step, against the oracle. The kernels read the per-unit counters from the
device, the fused append's flags are cleared by each step's combine kernel and the combine
advances the counters, so the same captured launches see a growing cache (P:234 evict-on-exit)
every replay. Checked: every replay's outputs (<= 2e-3, R14) and, at the end, every record
buffer, the window and the counters bit-exact, plus the host mirror kept in step by
mstf_graph_step_commit."""
import math

import numpy as np
import pytest

import synth
from oracle import mustafar_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-3


@pytest.fixture(scope="module")
def M():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_22913_b200 import build as B
    B.build()
    from paper_2505_22913_b200 import mustafar
    return mustafar


def rel_err(o_gpu, o_ref):
    d = np.abs(o_gpu.astype(np.float64) - o_ref).max(axis=-1)
    n = np.abs(o_ref).max(axis=-1)
    return float((d / n).max())


@pytest.mark.parametrize("case", [
    # (batch, hq, hkv, T, keep, W, layers, steps)
    (2, 8, 2, 300, 39, 32, 3, 40),     # full window: every replay evicts into a record
    (1, 8, 1, 10, 39, 32, 2, 45),      # window filling for 22 replays, then evicting
    (2, 4, 4, 200, 64, 0, 2, 40),      # W = 0 (the new token is compressed directly), G = 1
    (1, 8, 1, 500, 26, 16, 2, 40),     # G = 8
])
def test_graph_replay_matches_oracle(M, case):
    B, hq, hkv, T, keep, W, L, steps = case
    U, G, d = B * hkv, hq // hkv, 128
    scale = 1 / math.sqrt(d)
    cap = T + steps + 1
    Ks = [synth.fp16_np((U, T + steps, d), synth.seed_for(30 + l, 0)) for l in range(L)]
    Vs = [synth.fp16_np((U, T + steps, d), synth.seed_for(30 + l, 1)) for l in range(L)]
    Qs = synth.fp16_np((steps, L, U, G, d), synth.seed_for(40, 2))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.float16)
    caches, oracles = [], []
    for l in range(L):
        c = M.MustafarCache(B, hq, hkv, d, keep, keep, W, cap)
        c.prune_compress_kv(dev(Ks[l][:, :T]), dev(Vs[l][:, :T]))
        oc = O.OracleCache(U, d, keep, keep, W, cap)
        oc.prefill(Ks[l][:, :T].view(np.uint16), Vs[l][:, :T].view(np.uint16))
        caches.append(c)
        oracles.append(oc)
    # one warm-up call per cache before capture (kernel attributes are set outside the graph)
    qb = [torch.empty(U, G, d, dtype=torch.float16, device="cuda") for _ in range(L)]
    kb = [torch.empty(U, d, dtype=torch.float16, device="cuda") for _ in range(L)]
    vb = [torch.empty(U, d, dtype=torch.float16, device="cuda") for _ in range(L)]
    ob = [torch.empty(U, G, d, dtype=torch.float32, device="cuda") for _ in range(L)]

    def load(i):
        for l in range(L):
            qb[l].copy_(dev(Qs[i, l]))
            kb[l].copy_(dev(Ks[l][:, T + i]))
            vb[l].copy_(dev(Vs[l][:, T + i]))

    # step 0 eagerly (also the warm-up), steps 1.. through the graph
    load(0)
    for l in range(L):
        caches[l].decode_step(kb[l], vb[l], qb[l], scale, out=ob[l])
    torch.cuda.synchronize()
    graph = None
    for i in range(steps):
        if i > 0:
            load(i)
            if graph is None:
                graph = M.DecodeGraph(caches, qb, kb, vb, ob, scale)
            graph.replay()
            torch.cuda.synchronize()
        for l in range(L):
            oracles[l].append(Ks[l][:, T + i].view(np.uint16), Vs[l][:, T + i].view(np.uint16))
            ref = O.attention(oracles[l], Qs[i, l].view(np.uint16), scale)
            err = rel_err(ob[l].cpu().numpy(), ref)
            assert err <= TOL, (case, i, l, err)
    for l in range(L):
        oc = oracles[l]
        assert caches[l].counts() == (oc.n_comp.tolist(), oc.n_win.tolist())
        b = caches[l].buffers()
        assert b["n_comp"].cpu().tolist() == oc.n_comp.tolist()
        assert b["n_win"].cpu().tolist() == oc.n_win.tolist()
        for u in range(U):
            n = int(oc.n_comp[u])
            for name, dt in (("bitmap_k", np.uint64), ("bitmap_v", np.uint64), ("values_k", np.uint16),
                             ("values_v", np.uint16), ("offsets_k", np.uint32), ("offsets_v", np.uint32)):
                assert np.array_equal(b[name][u, :n].cpu().numpy().view(dt), getattr(oc, name)[u, :n]), (l, u, name)


def test_graph_step_check_rejects_capacity_and_ragged(M):
    """The host-side guard: no replay past capacity; a ragged cache (whose decode step is not the
    counter-independent fused launch) cannot be captured."""
    import ctypes  # noqa: F401
    U, d = 2, 128
    K = torch.zeros(U, 40, d, dtype=torch.float16, device="cuda")
    c = M.MustafarCache(1, 2, 2, d, 39, 39, 32, 40 - 32 + 3)   # room for 3 evictions
    c.prune_compress_kv(K, K)
    L = M.lib()
    assert L.mstf_graph_step_check(c._h, 3) == 0
    assert L.mstf_graph_step_check(c._h, 4) == -4
    r = M.MustafarCache(1, 2, 2, d, 39, 39, 32, 40)
    r.prune_compress_kv(K, K, lengths=[40, 12])
    assert L.mstf_graph_step_check(r._h, 1) == -1
    with pytest.raises(M.MustafarError):
        M.DecodeGraph([r], [torch.zeros(U, 1, d, dtype=torch.float16, device="cuda")],
                      [K[:, 0].contiguous()], [K[:, 0].contiguous()],
                      [torch.empty(U, 1, d, device="cuda")])
