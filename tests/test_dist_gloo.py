"""Multi-rank orchestration of the bucket-range-sharded build and routed lookup
(paper_2508_11443_b200/dist.py) on CPU with the gloo backend, world size 2 and 3.

The per-rank compute steps (route, shard build, local lookup, unroute) are
supplied by an oracle-backed stand-in for the libhm kernels, so this checks the
host logic: global n, owner ranges, the all-to-all splits, the global space
bound and t1 agreement, the slot bases, and that the shards concatenated in
rank order equal the single-table oracle.
"""
import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from oracle import oracle as O
from workloads import gen

MASK40 = np.uint64((1 << 40) - 1)


def _owner_of(keys, n, seed, t1, world):
    c1 = O.derive(seed, 1, 0, t1)
    b = np.array([O.hash_(c1, int(k)) % n for k in keys], dtype=np.int64)
    return b, (b * world) // n


class OracleShard:
    def __init__(self, table, n, lo, hi, t1, seed):
        self.t, self.n, self.lo, self.hi, self.t1, self.seed = table, n, lo, hi, t1, seed
        self.base = 0


class OracleOps:
    """CPU stand-in for dist.GpuOps built on the (pinned) oracle primitives."""

    def route(self, keys, vals, n_global, seed, t1, world):
        k = keys.numpy().view(np.uint64)
        _, own = _owner_of(k, n_global, seed, t1, world)
        order = np.argsort(own, kind="stable")
        counts = np.bincount(own, minlength=world)
        return keys[order], vals[order], torch.from_numpy(counts.astype(np.int64))

    def build_shard(self, keys, vals, n_global, lo, hi, t1, seed):
        st, t = O.build_u64_shard(keys.numpy().view(np.uint64), vals.numpy().view(np.uint64), n_global, lo, hi, t1,
                                  seed)
        code = {"OK": 0, "DUPLICATE_KEY": 3, "SEED_EXHAUSTED": 4}[st]
        return OracleShard(t, n_global, lo, hi, t1, seed), t.S, code

    def route_queries(self, shard, q, world):
        qq = q.numpy().view(np.uint64)
        _, own = _owner_of(qq, shard.n, shard.seed, shard.t1, world)
        order = np.argsort(own, kind="stable")
        perm = np.empty(len(qq), np.int64)
        perm[order] = np.arange(len(qq))
        return q[order], torch.from_numpy(perm), torch.from_numpy(np.bincount(own, minlength=world).astype(np.int64))

    def lookup(self, shard, q):
        qq = q.numpy().view(np.uint64)
        soff, s, tt = O.decode_dir(shard.t.dir)
        c1 = O.derive(shard.seed, 1, 0, shard.t1)
        vals = np.zeros(len(qq), np.uint64)
        found = np.zeros(len(qq), np.uint8)
        for i, k in enumerate(qq):
            b = O.hash_(c1, int(k)) % shard.n
            lb = b - shard.lo
            assert 0 <= lb < shard.hi - shard.lo
            sb = int(s[lb])
            if sb == 0:
                continue
            j = int(soff[lb])
            if sb > 1:
                j += O.hash_(O.derive(shard.seed, 2, b, int(tt[lb])), int(k)) % (sb * sb)
            if int(shard.t.slots["key"][j]) == int(k):
                vals[i] = shard.t.slots["value"][j]
                found[i] = 1
        return torch.from_numpy(vals.view(np.int64)), torch.from_numpy(found)

    def unroute(self, vals_r, found_r, perm, out_vals, out_found):
        out_vals.copy_(vals_r[perm])
        out_found.copy_(found_r[perm])

    def set_base(self, shard, base):
        shard.base = base

    def free(self, shard):
        pass

    def export_shard(self, shard, nb, S_local, device):
        d = shard.t.dir.copy()
        d = (d & ~MASK40) | ((d & MASK40) + np.uint64(shard.base))
        sl = np.stack([shard.t.slots["key"], shard.t.slots["value"]], axis=1).reshape(-1)
        return torch.from_numpy(d.view(np.int64)), torch.from_numpy(np.ascontiguousarray(sl).view(np.int64))

    def assemble(self, dir_, slots, n, S, seed, t1):
        sl = slots.numpy().view(np.uint64).reshape(-1, 2)
        assert dir_.numel() == n and sl.shape[0] == S
        t = types.SimpleNamespace(dir=dir_.numpy().view(np.uint64).copy(),
                                  slots={"key": sl[:, 0].copy(), "value": sl[:, 1].copy()})
        return OracleShard(t, n, 0, n, t1, seed)


def _worker(rank, world, port, n, seed, nq, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2508_11443_b200 import dist
        lo_i, hi_i = rank * n // world, (rank + 1) * n // world
        keys = torch.from_numpy(gen.u64_keys(hi_i - lo_i, lo=lo_i).view(np.int64))
        vals = torch.from_numpy(gen.u64_values(hi_i - lo_i, lo=lo_i).view(np.int64))
        dm = dist.build_dist(keys, vals, seed=seed, ops=OracleOps())
        d = dm.shard.t.dir.copy()
        d = (d & ~MASK40) | ((d & MASK40) + np.uint64(dm.slot_base))
        qlo, qhi = rank * nq // world, (rank + 1) * nq // world
        qq, _, _ = gen.u64_queries(n, qhi - qlo, lo=qlo)
        ov, of = dist.lookup_dist(dm, torch.from_numpy(qq.view(np.int64)))
        # replicated mode: the all-gathered single table, local lookups
        rep = dist.replicate_dist(dm)
        rv, rf = dm.ops.lookup(rep, torch.from_numpy(qq.view(np.int64)))
        assert torch.equal(rv, ov) and torch.equal(rf, of)
        out = (rank, dm.lo, dm.hi, dm.t1, d, dm.shard.t.slots.copy(), ov.numpy().view(np.uint64).copy(), of.numpy().copy(),
               rep.t.dir, rep.t.slots["key"])
        q.put(out)
    finally:
        tdist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# (2, 8, 167) and (2, 7, 247) need a level-1 redraw (t1 = 1): the global bound must be agreed
@pytest.mark.parametrize("world,n,seed", [(2, 3000, 0), (2, 7, 1), (3, 1001, 5), (2, 8, 167), (2, 7, 247)])
def test_sharded_build_equals_single_table(world, n, seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    nq = 600
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, seed, nq, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    t = O.build_u64(gen.u64_keys(n), gen.u64_values(n), seed)
    assert all(r[3] == int(t.header["t1"]) for r in res)
    assert [r[1] for r in res] == [-(-r * n // world) for r in range(world)]
    assert np.array_equal(np.concatenate([r[4] for r in res]), t.dir)
    assert np.concatenate([r[5] for r in res]).tobytes() == t.slots.tobytes()
    qq, _, _ = gen.u64_queries(n, nq)
    ov, of = O.lookup_u64(t, qq)
    assert np.array_equal(np.concatenate([r[6] for r in res]), ov)
    assert np.array_equal(np.concatenate([r[7] for r in res]), of)
    for r in res:  # every rank holds the whole single table after replicate_dist
        assert np.array_equal(r[8], t.dir) and np.array_equal(r[9], t.slots["key"])
