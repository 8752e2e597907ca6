"""Multi-GPU bucket-range sharding.

One process per GPU.  Rank r owns level-1 buckets [lo_r, lo_{r+1}) with
lo_r = ceil(r*n/G) (owner(b) = floor(b*G/n)), where n is the GLOBAL key count
(the level-1 modulus, R3).  The exchange between the route kernel and the
shard build is an all-to-all over torch.distributed (NCCL on GPUs, gloo in the
CPU tests); this module is plumbing only — every computation is a libhm
kernel, reached through an `ops` object (`GpuOps` here; the CPU tests pass an
oracle-backed stand-in to check the orchestration itself).

Build (all ranks, collectively):
  1. n = allreduce(n_local)                                   (C1)
  2. for t1 = 0, 1, ...: route (key, value) by owner rank,     (K7)
     exchange counts then payload (all_to_all)                  (C2)
     build the local shard with level-1 attempt t1              (K2-K5)
     S = allreduce(S_r); stop at the first t1 with S <= 4n      (C3, R7)
  3. allreduce the shard status so every rank raises the same error
  4. slot base of rank r = sum_{q<r} S_q (allgather)             (C3)
Lookup: route queries by owner, all_to_all, local lookup, all_to_all back,
unroute by the recorded permutation.
Replicated lookups: all-gather the exported shards into the single table on
every rank (hm_assemble_u64), then local lookups without an exchange.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as tdist

from . import hm as _hm


def bucket_range(rank: int, world: int, n: int):
    """[lo, hi) of the level-1 buckets owned by `rank` (owner(b) = floor(b*G/n)),
    hm_dist_bucket_range."""
    return _hm.dist_bucket_range(n, world, rank)


class GpuOps:
    """The libhm kernels behind the orchestration."""

    def route(self, keys, vals, n_global, seed, t1, world):
        sk = torch.empty_like(keys)
        sv = torch.empty_like(vals)
        counts = torch.zeros(world, dtype=torch.int64, device=keys.device)
        _hm.route_u64(keys, vals, n_global, seed, t1, world, sk, sv, counts)
        return sk, sv, counts

    def build_shard(self, keys, vals, n_global, lo, hi, t1, seed):
        try:
            m, S = _hm.build_u64_shard(keys, vals, n_global, lo, hi, t1, seed)
            return m, S, 0
        except _hm.HMError as e:
            return None, 0, e.code

    def route_queries(self, shard, q, world):
        sq = torch.empty_like(q)
        perm = torch.empty_like(q)
        counts = torch.zeros(world, dtype=torch.int64, device=q.device)
        shard.route_queries(q, world, sq, perm, counts)
        return sq, perm, counts

    def lookup(self, shard, q):
        return shard.lookup(q)

    def unroute(self, vals_r, found_r, perm, out_vals, out_found):
        _hm.unroute_u64(vals_r, found_r, perm, out_vals, out_found)

    def set_base(self, shard, base):
        shard.set_base(base)

    def free(self, shard):
        if shard is not None:
            shard.free()

    def export_shard(self, shard, nb, S_local, device):
        d = torch.empty(max(nb, 1), dtype=torch.int64, device=device)
        sl = torch.empty(max(2 * S_local, 2), dtype=torch.int64, device=device)
        if shard is not None:
            shard.export_to(d, sl)
        return d[:nb], sl[: 2 * S_local]

    def assemble(self, dir_, slots, n, S, seed, t1):
        return _hm.HashMap.assemble_u64(dir_, slots, n, S, seed, t1)


@dataclass
class DistMap:
    shard: object
    n_global: int
    lo: int
    hi: int
    t1: int
    S_local: int
    slot_base: int
    S_total: int
    world: int
    rank: int
    ops: object
    group: object = None
    seed: int = 0
    S_all: tuple = ()


def _exchange_counts(in_counts, group, device):
    """How many elements every rank sends here (all_to_all of the split sizes)."""
    cin = torch.tensor(in_counts, dtype=torch.int64, device=device)
    cout = torch.empty_like(cin)
    tdist.all_to_all_single(cout, cin, group=group)
    return [int(x) for x in cout.tolist()]


def _all_to_all_v(send, in_counts, group, device, out_counts=None):
    """Variable all-to-all of a 1-D tensor grouped by destination rank."""
    if out_counts is None:
        out_counts = _exchange_counts(in_counts, group, device)
    recv = torch.empty(sum(out_counts), dtype=send.dtype, device=send.device)
    tdist.all_to_all_single(recv, send, out_counts, list(in_counts), group=group)
    return recv, out_counts


def build_dist(keys, vals, seed: int = 0, ops=None, group=None) -> DistMap:
    """Collective build of a bucket-range-sharded FKS table."""
    ops = ops or GpuOps()
    world = tdist.get_world_size(group)
    rank = tdist.get_rank(group)
    dev = keys.device
    cnt = torch.tensor([keys.numel()], dtype=torch.int64, device=dev)
    tdist.all_reduce(cnt, group=group)
    n = int(cnt.item())
    if n == 0:
        raise _hm.HMError(2, "global key set is empty")
    lo, hi = bucket_range(rank, world, n)
    t1 = 0
    while True:
        sk, sv, counts = ops.route(keys, vals, n, seed, t1, world)
        in_counts = [int(x) for x in counts.tolist()]
        rk, out_counts = _all_to_all_v(sk, in_counts, group, dev)
        rv, _ = _all_to_all_v(sv, in_counts, group, dev, out_counts)  # (same splits)
        shard, S_local, code = ops.build_shard(rk, rv, n, lo, hi, t1, seed)
        # agree on the outcome: the space bound is global (R7), errors are global;
        # the decision itself is libhm's (hm_dist_decide, shared with hm_build_u64_dist)
        red = torch.tensor([S_local, code], dtype=torch.int64, device=dev)
        tdist.all_reduce(red[:1], group=group)
        tdist.all_reduce(red[1:], op=tdist.ReduceOp.MAX, group=group)
        S_total, code = int(red[0].item()), int(red[1].item())
        d, t1_next = _hm.dist_decide(n, t1, S_total, code)
        if d == 0:
            break
        ops.free(shard)
        if d != _hm.DIST_REDRAW:
            raise _hm.HMError(d, f"sharded build failed at t1={t1} (max status over ranks)")
        t1 = t1_next
    allS = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    tdist.all_gather(allS, torch.tensor([S_local], dtype=torch.int64, device=dev), group=group)
    base = _hm.dist_slot_base([int(x.item()) for x in allS], rank)
    ops.set_base(shard, base)
    return DistMap(shard, n, lo, hi, t1, S_local, base, S_total, world, rank, ops, group, seed,
                   tuple(int(x.item()) for x in allS))


def lookup_dist(dm: DistMap, q, out_vals=None, out_found=None):
    """Collective lookup: every rank passes its own queries, gets its own answers
    (written into out_vals / out_found when given)."""
    ops, group, world = dm.ops, dm.group, dm.world
    dev = q.device
    sq, perm, counts = ops.route_queries(dm.shard, q, world)
    in_counts = [int(x) for x in counts.tolist()]
    rq, out_counts = _all_to_all_v(sq, in_counts, group, dev)
    v, f = ops.lookup(dm.shard, rq)
    # results travel back along the reverse splits
    back_v = torch.empty(sum(in_counts), dtype=v.dtype, device=dev)
    tdist.all_to_all_single(back_v, v, in_counts, out_counts, group=group)
    back_f = torch.empty(sum(in_counts), dtype=f.dtype, device=dev)
    tdist.all_to_all_single(back_f, f, in_counts, out_counts, group=group)
    out_v = torch.empty_like(q) if out_vals is None else out_vals
    out_f = torch.empty(q.numel(), dtype=torch.uint8, device=dev) if out_found is None else out_found
    ops.unroute(back_v, back_f, perm, out_v, out_f)
    return out_v, out_f


def _all_gather_v(x, sizes, group):
    """All-gather of 1-D pieces of different lengths (padded to the largest)."""
    world = len(sizes)
    mx = max(max(sizes), 1)
    pad = torch.zeros(mx, dtype=x.dtype, device=x.device)
    pad[: x.numel()] = x
    parts = [torch.empty_like(pad) for _ in range(world)]
    tdist.all_gather(parts, pad, group=group)
    return torch.cat([p[:n] for p, n in zip(parts, sizes)])


def replicate_dist(dm: DistMap):
    """Replicated-lookup mode: every rank receives
    all shards (all-gather of the exported directories, whose soff are
    global, and of the slots) and assembles the single table, so lookups are
    local with no exchange.  Returns that map (a HashMap on this rank's GPU);
    the shards stay as they are.  Costs 8 + 16*S/n bytes per key per rank."""
    ops, group, world = dm.ops, dm.group, dm.world
    nb_all = [hi - lo for lo, hi in (bucket_range(r, world, dm.n_global) for r in range(world))]
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")
    d, sl = ops.export_shard(dm.shard, dm.hi - dm.lo, dm.S_local, dev)
    full_dir = _all_gather_v(d, nb_all, group)
    full_slots = _all_gather_v(sl, [2 * x for x in dm.S_all], group)
    return ops.assemble(full_dir, full_slots, dm.n_global, dm.S_total, dm.seed, dm.t1)


def free_dist(dm: DistMap):
    dm.ops.free(dm.shard)
    dm.shard = None
