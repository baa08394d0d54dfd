"""Ownership and halo rules of the partitioned multi-GPU evaluation
(fse_dist_rules.h via fse_dist_owner / fse_dist_masks), checked on the CPU by
brute force, and the halo exchange itself between two gloo processes
(world_size 2): every rank ends with exactly the sources its slab's spread
tiles and its owned targets' real-space neighbourhoods need, and every target
is shipped to each slab that holds part of its quadrature support.

The brute-force references: a source is needed by rank d when its support
[i0, i0 + P) (the C oracle's i0, ewald.cpp:33-51) meets d's x-planes, or when
some target owned by d lies within rc of it."""
import os
import socket

import numpy as np
import pytest


def slabs(Mt, G):
    nxs = ((Mt + G - 1) // G + 7) // 8 * 8 if G > 1 else Mt
    return nxs, [(min(d * nxs, Mt), max(0, min(nxs, Mt - min(d * nxs, Mt)))) for d in range(G)]


def check_rules(fse, oracle, args, G, pos, tgt):
    cfg = fse.make_config(*args)
    ocfg = oracle.make_config(*args)
    P = cfg.P
    nxs, sl = slabs(cfg.Mtilde, G)
    own_s = fse.dist_owner(cfg, G, pos)
    own_t = fse.dist_owner(cfg, G, tgt)
    ms = fse.dist_masks(cfg, G, pos, False)
    mt = fse.dist_masks(cfg, G, tgt, True)
    assert own_s.min() >= 0 and own_s.max() < G
    assert np.all((ms >> own_s.astype(np.uint32)) & 1) and np.all((mt >> own_t.astype(np.uint32)) & 1)
    i0s = oracle.support_index(ocfg, pos)[:, 0]
    i0t = oracle.support_index(ocfg, tgt)[:, 0]
    # owner = slab holding the support centre plane i0 + P/2
    assert np.array_equal(own_s, np.minimum((i0s + P // 2) // nxs, G - 1))
    for d, (lo, n) in enumerate(sl):
        hit_s = (n > 0) & (i0s < lo + n) & (i0s + P > lo)
        hit_t = (n > 0) & (i0t < lo + n) & (i0t + P > lo)
        bit_s = ((ms >> d) & 1).astype(bool)
        bit_t = ((mt >> d) & 1).astype(bool)
        assert np.all(bit_s[hit_s])                         # spread supports
        assert np.array_equal(bit_t, hit_t | (own_t == d))  # quadrature shares
        xt = tgt[own_t == d, 0]
        if xt.size:
            xs = np.sort(xt)
            k = np.searchsorted(xs, pos[:, 0])
            near = np.zeros(pos.shape[0], bool)
            for kk in (k - 1, k):
                ok = (kk >= 0) & (kk < xs.size)
                near[ok] |= np.abs(xs[kk[ok]] - pos[ok, 0]) <= cfg.rc
            assert np.all(bit_s[near])                      # real-space neighbours


@pytest.mark.parametrize("G", [1, 2, 3, 5, 8, 16])
@pytest.mark.parametrize("args", [(1.0, 12.0, 0.25, 48, 16), (1.0, 110.0, 0.045, 288, 24),
                                  (1.0, 20.0, 0.15, 56, 16)])
def test_rules_cover_the_halos(fse, oracle, rng, G, args):
    pos = rng.uniform(0, 1, (20000, 3))
    tgt = rng.uniform(0, 1, (5000, 3))
    check_rules(fse, oracle, args, G, pos, tgt)
    check_rules(fse, oracle, args, G, pos, pos)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as td

    import paper_1607_04808_b200 as fse
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = fse.make_config(1.0, 40.0, 0.1, 64, 16)
        rng = np.random.default_rng(11)  # every rank draws the same system ...
        pos = rng.uniform(0, 1, (6000, 3))
        st = rng.standard_normal((6000, 3))
        owner = fse.dist_owner(cfg, world, pos)
        mine = np.nonzero(owner == rank)[0]          # ... and keeps only what it owns
        ms = fse.dist_masks(cfg, world, pos[mine], False)
        # counts, then the ghost payloads (global index, position, strength), as the
        # device engine's pack step does, through gloo
        send = [mine[((ms >> d) & 1).astype(bool)] if d != rank else mine[:0]
                for d in range(world)]
        cnt = torch.tensor([len(x) for x in send], dtype=torch.int64)
        rcnt = torch.zeros(world, dtype=torch.int64)
        td.all_to_all_single(rcnt, cnt)
        payload = torch.tensor(np.concatenate([np.column_stack([i, pos[i], st[i]])
                                               for i in send]), dtype=torch.float64)
        recv = torch.zeros((int(rcnt.sum()), 7), dtype=torch.float64)
        td.all_to_all_single(recv, payload, [int(x) for x in rcnt], [int(x) for x in cnt])
        ghosts = recv.numpy()
        local = np.concatenate([mine, ghosts[:, 0].astype(np.int64)])
        assert np.array_equal(pos[ghosts[:, 0].astype(np.int64)], ghosts[:, 1:4])
        assert np.array_equal(st[ghosts[:, 0].astype(np.int64)], ghosts[:, 4:7])
        # what this rank needs, by brute force
        nxs = ((cfg.Mtilde + world - 1) // world + 7) // 8 * 8
        lo, n = rank * nxs, min(nxs, cfg.Mtilde - rank * nxs)
        s = (pos[:, 0] + cfg.deltaL / 2) / cfg.h
        i0 = np.ceil(s - cfg.P / 2).astype(np.int64)
        need = (i0 < lo + n) & (i0 + cfg.P > lo)
        xt = pos[mine, 0]
        need |= (pos[:, 0] >= xt.min() - cfg.rc) & (pos[:, 0] <= xt.max() + cfg.rc)
        have = np.zeros(pos.shape[0], bool)
        have[local] = True
        assert len(np.unique(local)) == len(local)       # no duplicates
        assert np.all(have[need])
        q.put((rank, len(mine), len(local)))
    finally:
        td.destroy_process_group()


def test_gloo_two_rank_halo_exchange():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
    assert all(p.exitcode == 0 for p in ps)
    res = sorted(q.get() for _ in range(2))
    assert sum(r[1] for r in res) == 6000       # owners partition the points
    assert all(r[2] < 6000 for r in res)        # and a rank holds only part of them
