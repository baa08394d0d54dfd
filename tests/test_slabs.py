"""z-slab decomposition (paper_1607_04808_b200/slabs.py).

CPU (no GPU needed): the slab partition math of fse_cuda_slab_info and the
block all-to-all / sum of TorchExchange over a world_size-2 gloo group.
GPU: the G-slab pipeline run as G virtual ranks in sequence on one device
(no kernel waits on another rank) equals the one-GPU total_sum.
"""
import os
import socket

import numpy as np
import pytest

from conftest import rel_max


def _cfg(fse, M=40, P=16, xi=15.0, rc=0.25):
    return fse.make_config(1.0, xi, rc, M, P)


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("M,P", [(40, 16), (48, 24), (88, 20)])
def test_slab_partition(fse, G, M, P):
    cfg = _cfg(fse, M=M, P=P)
    Mt, D = cfg.Mtilde, 2 * cfg.Mtilde
    xs, ks = [], []
    for r in range(G):
        inf = fse.api.slab_info(cfg, 0, r, G)
        assert inf.nxs % 8 == 0 or G == 1
        assert 0 <= inf.nx <= inf.nxs and 0 <= inf.nky <= inf.nkys
        xs += list(range(inf.x_lo, inf.x_lo + inf.nx))
        ks += list(range(inf.ky_lo, inf.ky_lo + inf.nky))
        assert inf.block_complex == 3 * inf.nxs * inf.nkys * (D // 2 + 1)
    assert xs == list(range(Mt)) and ks == list(range(D))


def test_slab_partition_rejects(fse):
    cfg = _cfg(fse, M=40, P=32)  # P + 7 > 32: no tensor-core quadrature variant
    with pytest.raises(fse.InvalidArgument):
        fse.api.slab_info(cfg, 0, 0, 2)
    fse.api.slab_info(cfg, 0, 0, 1)  # one slab is the plain path
    with pytest.raises(fse.InvalidArgument):
        fse.api.slab_info(_cfg(fse), 0, 2, 2)


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1607_04808_b200.slabs import TorchExchange
        ex = TorchExchange()
        blk = 5
        send = torch.tensor([100.0 * rank + 10.0 * s + j for s in range(world)
                             for j in range(blk)], dtype=torch.float64)
        recv = torch.full_like(send, -1.0)
        ex.all_to_all(send, recv)
        want = [100.0 * r + 10.0 * rank + j for r in range(world) for j in range(blk)]
        ok1 = recv.tolist() == want
        t = torch.arange(6, dtype=torch.float64) * (rank + 1)
        ex.all_reduce_sum(t)
        ok2 = t.tolist() == (torch.arange(6, dtype=torch.float64) * sum(range(1, world + 1))).tolist()
        q.put((rank, ok1, ok2))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_gloo(world):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert sorted(r for r, _, _ in res) == list(range(world))
    assert all(a and b for _, a, b in res), res


# ------------------------------------------------------------------ GPU
def _case(fse, ctx, rng, kind, n, args, distinct):
    L, xi, rc, M, P = args
    cfg = fse.make_config(L, xi, rc, M, P)
    pos = rng.uniform(0, L, (n, 3))
    st = rng.standard_normal((n, fse.strength_arity(kind)))
    tgt = rng.uniform(0, L, (n // 2, 3)) if distinct else pos
    g = ctx.precompute_mollified_green(int(fse.green_kind_for(kind)), cfg.Ltilde, cfg.Mtilde,
                                       cfg.sf)
    return cfg, fse.SourceSystem(pos, st, L), tgt, g


@pytest.mark.gpu
@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("G", [1, 2, 3])
@pytest.mark.parametrize("distinct", [False, True])
def test_slab_pipeline_matches_total_sum(fse, ctx, rng, kind, G, distinct):
    from paper_1607_04808_b200 import slabs
    cfg, s, tgt, g = _case(fse, ctx, rng, kind, 3000, (1.0, 15.28, 0.25, 40, 24), distinct)
    want = ctx.total_sum(s, kind, cfg, tgt, g)
    got = slabs.simulate(ctx, cfg, kind, s.positions, s.strengths, tgt, g, G,
                         targets_are_sources=not distinct)
    # same arithmetic per plane, only the order of the per-slab partial sums differs
    assert rel_max(got, want) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 5])
def test_slab_pipeline_uneven(fse, ctx, rng, G):
    """M~ not a multiple of 8 G, odd D/G: uneven slabs and ky blocks."""
    from paper_1607_04808_b200 import slabs
    cfg, s, tgt, g = _case(fse, ctx, rng, 0, 2000, (1.0, 12.0, 0.3, 37, 18), False)
    want = ctx.total_sum(s, 0, cfg, tgt, g)
    got = slabs.simulate(ctx, cfg, 0, s.positions, s.strengths, tgt, g, G,
                         targets_are_sources=True)
    assert rel_max(got, want) <= 1e-12
    peer = slabs.simulate(ctx, cfg, 0, s.positions, s.strengths, tgt, g, G,
                          targets_are_sources=True, peers=True)
    assert np.array_equal(peer, got)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("G", [2, 3, 4])
def test_peer_exchange_equals_all_to_all(fse, ctx, rng, kind, G):
    """Peer-direct exchange (fse_cuda_slab_forward_peers / _scale_peers: every
    block stored straight into its owner's buffer) is bit-identical to the
    all-to-all path: same kernels, same arithmetic, only the destinations of
    the stores differ."""
    from paper_1607_04808_b200 import slabs
    cfg, s, tgt, g = _case(fse, ctx, rng, kind, 2500, (1.0, 15.28, 0.25, 40, 24), True)
    a2a = slabs.simulate(ctx, cfg, kind, s.positions, s.strengths, tgt, g, G,
                         targets_are_sources=False)
    peer = slabs.simulate(ctx, cfg, kind, s.positions, s.strengths, tgt, g, G,
                          targets_are_sources=False, peers=True)
    assert np.array_equal(peer, a2a)
    want = ctx.total_sum(s, kind, cfg, tgt, g)
    assert rel_max(peer, want) <= 1e-12


@pytest.mark.gpu
def test_peer_exchange_rejects_bad_tables(fse, ctx, rng):
    cfg, s, tgt, g = _case(fse, ctx, rng, 0, 500, (1.0, 15.28, 0.25, 40, 24), False)
    with pytest.raises(fse.InvalidArgument):
        ctx.slab_forward_peers(cfg, 0, 0, 0, 0, 0, 17, [1] * 17)  # > 16 slabs
    with pytest.raises(fse.InvalidArgument):
        ctx.slab_forward_peers(cfg, 0, 0, 0, 0, 0, 2, [0, 0])  # null peer buffers
