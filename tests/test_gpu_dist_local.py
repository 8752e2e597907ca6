"""The multi-GPU path on one GPU: every rank's steps of the
bucket-range-sharded build and the routed lookup run through the real libhm
kernels (route, shard build with b_lo > 0, slot base, query routing, local
lookup, unroute), with the all-to-all exchanges done by concatenation in
this process.  The shards concatenated in rank order must equal the
single-table oracle byte for byte, and routed lookups must equal the oracle's.
A second test runs dist.build_dist / lookup_dist through NCCL itself with a
one-rank process group (the exact code bench.py runs at N > 1).
"""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from workloads import gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint64) if t.dtype == torch.int64 else t.cpu().numpy()


def _split(x, counts):
    out, o = [], 0
    for c in counts:
        out.append(x[o:o + c])
        o += c
    return out


@pytest.mark.parametrize("world,n,seed", [(2, 70_001, 0), (3, 100_000, 5), (4, 1 << 16, 2), (5, 3_000, 1)])
def test_sharded_build_and_routed_lookup_on_one_gpu(world, n, seed):
    from paper_2508_11443_b200 import dist
    ops = dist.GpuOps()
    keys, vals = gen.u64_keys(n), gen.u64_values(n)
    ot = O.build_u64(keys, vals, seed)
    # rank r holds keys[r n / W, (r + 1) n / W)
    cut = [r * n // world for r in range(world + 1)]
    kr = [dev(keys[cut[r]:cut[r + 1]]) for r in range(world)]
    vr = [dev(vals[cut[r]:cut[r + 1]]) for r in range(world)]
    for t1 in range(16):
        routed = [ops.route(kr[r], vr[r], n, seed, t1, world) for r in range(world)]
        parts_k = [_split(sk, [int(c) for c in cnt.tolist()]) for sk, _, cnt in routed]
        parts_v = [_split(sv, [int(c) for c in cnt.tolist()]) for _, sv, cnt in routed]
        shards = []
        for d in range(world):
            lo, hi = dist.bucket_range(d, world, n)
            rk = torch.cat([parts_k[r][d] for r in range(world)])
            rv = torch.cat([parts_v[r][d] for r in range(world)])
            shards.append(ops.build_shard(rk, rv, n, lo, hi, t1, seed))
        assert all(code == 0 for _, _, code in shards)
        if sum(S for _, S, _ in shards) <= 4 * n:
            break
        for m, _, _ in shards:
            ops.free(m)
    assert t1 == int(ot.header["t1"])
    base = 0
    for m, S, _ in shards:
        ops.set_base(m, base)
        base += S
    assert base == ot.S
    dirs, slots = [], []
    for m, _, _ in shards:
        d, sl, _ = m.export()
        dirs.append(d)
        slots.append(sl)
    assert np.concatenate(dirs).tobytes() == ot.dir.tobytes()
    assert np.concatenate(slots).tobytes() == ot.slots.tobytes()
    # replicated mode: the shards' device exports, concatenated, assembled into
    # the single table (hm_assemble_u64) — identical to the oracle's
    dd, ss = [], []
    for d_ in range(world):
        lo, hi = dist.bucket_range(d_, world, n)
        a, b = ops.export_shard(shards[d_][0], hi - lo, shards[d_][1], torch.device("cuda"))
        dd.append(a)
        ss.append(b)
    rep = ops.assemble(torch.cat(dd), torch.cat(ss), n, ot.S, seed, t1)
    rd, rs, _ = rep.export()
    assert rd.tobytes() == ot.dir.tobytes() and rs.tobytes() == ot.slots.tobytes()
    # routed lookups: rank r asks its own queries
    q, _, _ = gen.u64_queries(n, 3 * n)
    ov, of = O.lookup_u64(ot, q)
    qcut = [r * len(q) // world for r in range(world + 1)]
    qs = [dev(q[qcut[r]:qcut[r + 1]]) for r in range(world)]
    rq = [ops.route_queries(shards[0][0], qs[r], world) for r in range(world)]
    parts_q = [_split(sq, [int(c) for c in cnt.tolist()]) for sq, _, cnt in rq]
    answers = []
    for d in range(world):
        v, f = ops.lookup(shards[d][0], torch.cat([parts_q[r][d] for r in range(world)]))
        sizes = [len(parts_q[r][d]) for r in range(world)]
        answers.append((_split(v, sizes), _split(f, sizes)))
    for r in range(world):
        back_v = torch.cat([answers[d][0][r] for d in range(world)])
        back_f = torch.cat([answers[d][1][r] for d in range(world)])
        out_v = torch.empty_like(qs[r])
        out_f = torch.empty(qs[r].numel(), dtype=torch.uint8, device="cuda")
        ops.unroute(back_v, back_f, rq[r][1], out_v, out_f)
        assert np.array_equal(host(out_v), ov[qcut[r]:qcut[r + 1]])
        assert np.array_equal(host(out_f), of[qcut[r]:qcut[r + 1]])
    rv, rf = rep.lookup(dev(q))
    assert np.array_equal(host(rv), ov) and np.array_equal(host(rf), of)
    rep.free()
    for m, _, _ in shards:
        ops.free(m)


def test_assemble_from_export_and_rejects_non_tables():
    """hm_assemble_u64 on a host export of a built map gives the same table and
    the same lookups (the compact directory re-derived, singleton tags included);
    a directory whose offsets do not add up is refused."""
    from paper_2508_11443_b200 import hm
    n = 200_003
    keys, vals = gen.u64_keys(n), gen.u64_values(n)
    m = hm.HashMap.build_u64(dev(keys), dev(vals), seed=6)
    d, sl, _ = m.export()
    inf = m.info()
    a = hm.HashMap.assemble_u64(d, sl, n, inf.S, 6, inf.t1)
    d2, sl2, _ = a.export()
    assert d2.tobytes() == d.tobytes() and sl2.tobytes() == sl.tobytes()
    assert a.header_bytes() == m.header_bytes()
    q, _, _ = gen.u64_queries(n, 3 * n)
    v1, f1 = m.lookup(dev(q))
    v2, f2 = a.lookup(dev(q))
    assert torch.equal(v1, v2) and torch.equal(f1, f2)
    full = hm.HashMap.assemble_u64(d, sl, n, inf.S, 6, inf.t1, flags=hm.FLAG_FULL_DIRECTORY)
    v3, f3 = full.lookup(dev(q))
    assert torch.equal(v1, v3) and torch.equal(f1, f3)
    for x in (a, full):
        x.free()
    bad = d.copy()
    bad[n // 2] += np.uint64(1)  # an soff off by one
    with pytest.raises(hm.HMError) as e:
        hm.HashMap.assemble_u64(bad, sl, n, inf.S, 6, inf.t1)
    assert e.value.name == "INVALID_ARG"
    with pytest.raises(hm.HMError) as e:
        hm.HashMap.assemble_u64(d, sl, n, inf.S - 1, 6, inf.t1)
    assert e.value.name == "INVALID_ARG"
    m.free()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_dist_build_and_lookup_through_nccl_one_rank():
    import torch.distributed as tdist

    from paper_2508_11443_b200 import dist
    torch.cuda.set_device(0)
    tdist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", world_size=1, rank=0,
                             device_id=torch.device("cuda", 0))
    try:
        n = 100_003
        keys, vals = gen.u64_keys(n), gen.u64_values(n)
        ot = O.build_u64(keys, vals, 3)
        dm = dist.build_dist(dev(keys), dev(vals), seed=3)
        assert dm.S_total == ot.S and dm.t1 == int(ot.header["t1"])
        d, sl, _ = dm.shard.export()
        assert d.tobytes() == ot.dir.tobytes() and sl.tobytes() == ot.slots.tobytes()
        q, _, _ = gen.u64_queries(n, 2 * n)
        v, f = dist.lookup_dist(dm, dev(q))
        ov, of = O.lookup_u64(ot, q)
        assert np.array_equal(host(v), ov) and np.array_equal(host(f), of)
        rep = dist.replicate_dist(dm)
        rv, rf = rep.lookup(dev(q))
        assert np.array_equal(host(rv), ov) and np.array_equal(host(rf), of)
        rep.free()
        dist.free_dist(dm)
        # the same through the single C calls over the process group's communicator
        from paper_2508_11443_b200 import hm
        comm = tdist.distributed_c10d._get_default_group()._get_backend(torch.device("cuda", 0))._comm_ptr()
        m = hm.build_u64_dist(dev(keys), dev(vals), comm, seed=3)
        d, sl, _ = m.export()
        assert d.tobytes() == ot.dir.tobytes() and sl.tobytes() == ot.slots.tobytes()
        v, f = hm.lookup_u64_dist(m, dev(q), comm)
        assert np.array_equal(host(v), ov) and np.array_equal(host(f), of)
        dup = keys.copy()
        dup[5] = dup[99]
        with pytest.raises(hm.HMError) as e:
            hm.build_u64_dist(dev(dup), dev(vals), comm)
        assert e.value.name == "DUPLICATE_KEY"
        m.free()
        # NEXT-2: the route kernel storing straight into the owner's NCCL
        # window (here the owner is this rank): the same table
        m = hm.build_u64_dist(dev(keys), dev(vals), comm, seed=3, flags=hm.FLAG_FUSED_EXCHANGE)
        d, sl, _ = m.export()
        assert d.tobytes() == ot.dir.tobytes() and sl.tobytes() == ot.slots.tobytes()
        v, f = hm.lookup_u64_dist(m, dev(q), comm)
        assert np.array_equal(host(v), ov) and np.array_equal(host(f), of)
        m.free()
        with pytest.raises(hm.HMError) as e:
            hm.build_u64_dist(dev(dup), dev(vals), comm, flags=hm.FLAG_FUSED_EXCHANGE)
        assert e.value.name == "DUPLICATE_KEY"
    finally:
        tdist.destroy_process_group()
