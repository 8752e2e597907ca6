#!/usr/bin/env python
"""bench.py — FKS build + batched lookup on B200 (BASELINE.json metric).

One step = one pass of the whole hot path over one batch:
build the FKS table from n device-resident (key, value) pairs (level-1 hash,
partition, per-bucket histogram/scans, level-2 seed search, table write) and
answer n lookups at 50% hit rate (PAPER.md:903-915 workload shape, recipe in
DESIGN.md §3), then free the table.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N=1: BASELINE.json configs[1] — 2^26 random distinct u64 keys with u64
values, 2^26 lookups at 50% hit.  N>1: one process per GPU; without
torchrun's WORLD_SIZE in the environment, bench.py re-launches itself through
torch.distributed.run with N ranks (and refuses to run on fewer GPUs).  Every
rank holds 2^26 keys and 2^26 queries of one global table of N*2^26 keys
(N=8: configs[3]'s 2^29), bucket-range sharded by hm_build_u64_dist /
hm_lookup_u64_dist over the process group's NCCL communicator (weak scaling,
DESIGN.md §7).  Inputs are larger than L2 (126 MB): no flush between steps.

`value` = keys processed per second (one key = one key built + one query
answered) over all ranks, timed with CUDA events between barriers, max over
ranks.  The JSON line also carries the separate build and lookup rates, the
roofline of the dominant kernel (live CUDA-event timing of every libhm launch,
hm_profile_*), the other BASELINE configs measured after the timed region
(`configs`: C1, C3 string keys, C5 lookup-heavy; each with its roofline
fraction), the oracle's CPU baseline (one thread and all host threads), the
end-to-end rate through the C-ABI with pinned host buffers, the clocks seen
during the timed region and the number of libhm kernel launches.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FKS build Mkeys/s and lookup Mqueries/s, u64 & string keys, 1–8 B200"
LOG2N = 26
# SURVEY §8(d) byte models (algorithmic bytes per unit)
LOOKUP_BYTES_PER_QUERY = 8 + 32 + 32 * (0.5 + 0.5 * (1 - 0.36787944117)) + 8 + 1  # 75.1 B
BUILD_BYTES_PER_KEY = 56.0  # read key+value 16, dir 8, slots 16*S/n (~32)
STR_BUILD_BYTES_PER_KEY = 156.0  # offsets 8 + bytes 34 + values 8 + dir 8 + 32 B slots * 2 + context copy 34
STR_LOOKUP_BYTES_PER_QUERY = 142.0  # offsets 8 + bytes 34 + dir 32 + slot 26.1 + ~32.5 hit bytes + 9


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region (200 ms)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev = dev
        self.lines = []
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ CPU oracle

def host_info():
    model, mem = None, None
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                model = l.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        for l in open("/proc/meminfo"):
            if l.startswith("MemTotal"):
                mem = round(int(l.split()[1]) / 2**20, 1)
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "mem_gib": mem}


def oracle_pass(k, v, q, threads: int):
    """One oracle build + lookup pass: one thread (or_build_u64) or `threads`
    threads (or_build_u64_mt: level-1 bucket ranges per thread; the lookups
    split into `threads` slices, ctypes releases the GIL).  Returns
    (build seconds, lookup seconds)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O
    t0 = time.perf_counter()
    t = O.build_u64(k, v, 0) if threads == 1 else O.build_u64_mt(k, v, 0, threads)
    t1 = time.perf_counter()
    if threads == 1:
        O.lookup_u64(t, q)
    else:
        step = -(-len(q) // threads)
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda i: O.lookup_u64(t, q[i:i + step]), range(0, len(q), step)))
    t2 = time.perf_counter()
    del t
    return t1 - t0, t2 - t1


def cpu_baseline(log2n_sample: int = 24):
    """The oracle as it stands on a bounded sample of the same workload: all
    host threads (the value) and one thread (single_thread)."""
    from workloads import gen
    n = 1 << log2n_sample
    k, v = gen.u64_keys(n), gen.u64_values(n)
    q, _, _ = gen.u64_queries(n, n)
    T = os.cpu_count() or 1
    bt, lt = oracle_pass(k, v, q, T)
    b1, l1 = oracle_pass(k, v, q, 1)
    sample = f"2^{log2n_sample} keys built + 2^{log2n_sample} lookups (same recipe), one pass"
    return {"value": round(n / (bt + lt) / 1e6, 4), "unit": "Mkeys/s", "cores": T, "kind": "oracle",
            "sample": sample, "build_mkeys_s": round(n / bt / 1e6, 4), "lookup_mq_s": round(n / lt / 1e6, 4),
            "single_thread": {"value": round(n / (b1 + l1) / 1e6, 4), "cores": 1,
                              "build_mkeys_s": round(n / b1 / 1e6, 4), "lookup_mq_s": round(n / l1 / 1e6, 4)},
            "host": host_info()}


REF_LOG2 = 22


def config_dict(world):
    return {"workload": "configs[1]: 2^26 random distinct u64 keys + u64 values, build + 2^26 lookups at 50% hit"
            + (" per rank; global table of %d*2^26 keys bucket-range sharded over NCCL" % world if world > 1 else ""),
            "keys_per_gpu": 1 << LOG2N, "queries_per_gpu": 1 << LOG2N, "global_keys": world << LOG2N,
            "hit_rate": 0.5, "key_type": "u64", "value_type": "u64", "table_seed": 0,
            "seeds": {"SEED_K": 1, "SEED_Q": 2}, "parallelism": f"bucket-range shards x{world}" if world > 1 else "1 GPU",
            "l2": "inputs (512 MiB keys, 512 MiB values, 512 MiB queries) exceed the 126 MB L2; no flush"}


def run_reference(args):
    """--impl reference: the CPU oracle (plain C) on all host threads, each step
    one oracle pass over a bounded 2^22 sample of the config's workload (the
    per-key rate is the metric's unit).  Under torchrun only rank 0 runs."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return 0
    from workloads import gen
    n = 1 << REF_LOG2
    k, v = gen.u64_keys(n), gen.u64_values(n)
    q, _, _ = gen.u64_queries(n, n)
    T = os.cpu_count() or 1
    times = []
    for i in range(args.warmup + args.steps):
        bt, lt = oracle_pass(k, v, q, T)
        if i >= args.warmup:
            times.append(bt + lt)
    ms = 1e3 * statistics.mean(times)
    val = n / (ms / 1e3) / 1e6
    sample = (f"each step: one oracle pass (or_build_u64_mt + sliced or_lookup_u64, {T} host threads) over "
              f"2^{REF_LOG2} keys + 2^{REF_LOG2} lookups of the config's workload")
    cfg = config_dict(world)
    cfg["reference_sample"] = f"2^{REF_LOG2} keys + 2^{REF_LOG2} queries per step (bounded CPU sample)"
    out = {
        "impl": "reference", "metric": METRIC, "value": round(val, 4), "unit": "Mkeys/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic (workloads/gen.py recipe)",
        "config": cfg,
        "cpu_baseline": {"value": round(val, 4), "unit": "Mkeys/s", "cores": T, "kind": "oracle", "sample": sample,
                         "host": host_info()},
        "e2e": {"value": round(val, 4), "unit": "Mkeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return 0


# ------------------------------------------------------------------ launcher

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn(args) -> int:
    """N > 1 without torchrun: re-launch this script with N ranks (one per GPU)."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.stderr.write(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible; "
                         f"one rank per GPU needs {args.gpus}\n")
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ our path

def timed(fn, reps, warm=2):
    """Median device ms of fn() over reps (CUDA events on the current stream)."""
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def frac(units, ms, bpu, peak):
    return round(units * bpu / (ms / 1e3) / 1e9 / peak, 4)


def extra_configs(world, rank, dev, comm, peak, use_dist):
    """The other BASELINE configs, measured after the timed region (not part of
    `value`): C1 (2^16, launch-bound), C3 (2^24 strings, 4-64 bytes) and C5
    (2^30 lookups on a 2^27-key table; bucket-routed over the ranks for N>1)."""
    import torch

    from paper_2508_11443_b200 import hm
    from workloads import gen_cuda
    out = {}
    if world == 1:
        # C1: 2^16 keys, 2^16 queries
        n = 1 << 16
        k, v = gen_cuda.u64_keys(n)
        q, ev, ef = gen_cuda.u64_queries(n, n, with_expect=True)
        box = []

        def b1():
            m = hm.HashMap.build_u64(k, v)
            if box:
                box.pop().free()
            box.append(m)
        bms = timed(b1, 20)
        m = box[0]
        ov, of = torch.empty_like(q), torch.empty(n, dtype=torch.uint8, device=dev)
        lms = timed(lambda: m.lookup(q, ov, of), 20)
        ok = bool(torch.equal(ov, ev)) and bool(torch.equal(of, ef))
        m.free()
        out["C1"] = {"n": n, "build_ms": round(bms, 4), "lookup_ms": round(lms, 4), "correct": ok,
                     "build_mkeys_s": round(n / bms / 1e3, 1), "lookup_mq_s": round(n / lms / 1e3, 1),
                     "bound": "launch/latency (L2-resident)"}
        # C3: 2^24 strings of 4..64 bytes, 2^24 needles at 50% hit in their own context
        n = 1 << 24
        ctx, offs = gen_cuda.string_keys(n)
        vals = torch.arange(n, dtype=torch.int64, device=dev)
        box = []

        def b3():
            m = hm.HashMap.build_bytes(ctx, offs, vals)
            if box:
                box.pop().free()
            box.append(m)
        hm.profile_read()
        hm.profile_enable(True)
        bms = timed(b3, 5)
        bk = {a: round(b[1] / b[0], 4) for a, b in hm.profile_read().items()}
        m = box[0]
        qc, qo, ids = gen_cuda.string_queries(n, n)
        ov = torch.empty(n, dtype=torch.int64, device=dev)
        of = torch.empty(n, dtype=torch.uint8, device=dev)
        lms = timed(lambda: m.lookup_bytes(qc, qo, ov, of), 5)
        hm.profile_enable(False)
        lk = {a: round(b[1] / b[0], 4) for a, b in hm.profile_read().items() if a.startswith("k_lookup")}
        member = ids < n
        ok = bool(torch.equal(of.bool(), member)) and bool(torch.equal(ov[member], ids[member]))
        m.free()
        out["C3"] = {"n": n, "ctx_bytes": int(ctx.numel()), "build_ms": round(bms, 4), "lookup_ms": round(lms, 4),
                     "build_mkeys_s": round(n / bms / 1e3, 1), "lookup_mq_s": round(n / lms / 1e3, 1),
                     "build_roofline_frac": frac(n, bms, STR_BUILD_BYTES_PER_KEY, peak),
                     "lookup_roofline_frac": frac(n, lms, STR_LOOKUP_BYTES_PER_QUERY, peak),
                     "bytes_per_key": {"build": STR_BUILD_BYTES_PER_KEY, "lookup": STR_LOOKUP_BYTES_PER_QUERY},
                     "build_kernels_ms": bk, "lookup_kernels_ms": lk, "correct": ok}
        del ctx, offs, vals, qc, qo, ids, ov, of
        torch.cuda.empty_cache()
    # C5: 2^27-key table, 2^30 queries (per rank: 2^27/N keys, 2^30/N queries)
    n_glob, nq_glob = 1 << 27, 1 << 30
    n, nq = n_glob // world, nq_glob // world
    k, v = gen_cuda.u64_keys(n, lo=rank * n)
    chunk = min(nq, 1 << 28)
    q, ev, ef = gen_cuda.u64_queries(n_glob, chunk, lo=rank * nq, with_expect=True)
    ov = torch.empty(chunk, dtype=torch.int64, device=dev)
    of = torch.empty(chunk, dtype=torch.uint8, device=dev)
    if not use_dist:
        m = hm.HashMap.build_u64(k, v)
        look = lambda: [m.lookup(q, ov, of) for _ in range(nq // chunk)]  # noqa: E731
    else:
        m = hm.build_u64_dist(k, v, comm)
        look = lambda: [hm.lookup_u64_dist(m, q, comm, ov, of) for _ in range(nq // chunk)]  # noqa: E731
    lms = timed(look, 3, warm=1)
    ok = bool(torch.equal(ov, ev)) and bool(torch.equal(of, ef))
    m.free()
    out["C5"] = {"table_keys": n_glob, "queries": nq_glob, "lookup_ms": round(lms, 4),
                 "lookup_mq_s": round(nq_glob / lms / 1e3, 1),
                 "lookup_roofline_frac_per_gpu": frac(nq, lms, LOOKUP_BYTES_PER_QUERY, peak),
                 "routing": "bucket-routed all-to-all (hm_lookup_u64_dist)" if use_dist else "local",
                 "correct": ok, "timing": "rank-local CUDA events" if world > 1 else "CUDA events"}
    del k, v, q, ev, ef, ov, of
    torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch
    import torch.distributed as tdist

    from paper_2508_11443_b200 import hm
    from workloads import gen_cuda

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.stderr.write(f"bench.py --gpus {args.gpus} is running with WORLD_SIZE={world}: "
                         "one rank per GPU is required\n")
        return 2
    if torch.cuda.device_count() < world:
        sys.stderr.write(f"bench.py: {world} ranks but {torch.cuda.device_count()} CUDA device(s)\n")
        return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    use_dist = world > 1 or args.dist_path  # (--dist-path: the sharded C calls with one rank, a check of this path)
    if use_dist:
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
            os.environ["NCCL_DEBUG"] = "WARN"  # (no version banner ahead of the JSON line)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        # (NCCL prints its version banner on stdout when the communicator is
        # created: sent to stderr, so that stdout carries only the JSON line)
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            tdist.init_process_group("nccl", device_id=dev)
            tdist.barrier()
            comm = tdist.distributed_c10d._get_default_group()._get_backend(dev)._comm_ptr()
            torch.cuda.synchronize()
        finally:
            os.dup2(saved, 1)
            os.close(saved)

    def barrier():
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    n = 1 << LOG2N
    n_global = n * world
    keys, vals = gen_cuda.u64_keys(n, lo=rank * n)
    q, ev, ef = gen_cuda.u64_queries(n_global, n, lo=rank * n, with_expect=True)
    ov = torch.empty(n, dtype=torch.int64, device=dev)
    of = torch.empty(n, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    s_over_n = 2.0  # replaced by the table's actual S / n after the first step
    # N > 1: the fused route + exchange (NEXT-2) unless --no-fused-exchange;
    # a communicator that cannot register the symmetric window falls back to
    # route + grouped send/recv (decided on the first warm-up step, every rank
    # sees the same NCCL error)
    fused = use_dist and (args.fused_exchange or (world > 1 and not args.no_fused_exchange))
    dist_flags = hm.FLAG_FUSED_EXCHANGE if fused else 0
    fused_note = None

    def step(ev_b=None):
        nonlocal s_over_n
        if not use_dist:
            m = hm.HashMap.build_u64(keys, vals, seed=0)
        else:
            m = hm.build_u64_dist(keys, vals, comm, seed=0, flags=dist_flags)
        s_over_n = m.info().S / n
        if ev_b is not None:
            ev_b.record()
        if not use_dist:
            m.lookup(q, ov, of)
        else:
            hm.lookup_u64_dist(m, q, comm, ov, of)
        m.free()

    for i in range(args.warmup):
        if i == 0 and fused:
            try:
                step()
            except hm.HMError as e:
                fused, dist_flags, fused_note = False, 0, f"fused exchange unavailable ({e}); route + send/recv"
                barrier()
                step()
        else:
            step()
    barrier()
    # ---------------------------------------------------------------- timed
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    hm.profile_read()
    hm.profile_enable(True)
    l0 = hm.kernel_launches()
    barrier()
    e_start = torch.cuda.Event(enable_timing=True)
    e_end = torch.cuda.Event(enable_timing=True)
    marks = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
              torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    e_start.record()
    for (a, b, c) in marks:
        a.record()
        step(b)
        c.record()
    e_end.record()
    barrier()
    launches = hm.kernel_launches() - l0
    hm.profile_enable(False)
    kstats = hm.profile_read()
    clocks = clk.stop()
    total_ms = max_over_ranks(e_start.elapsed_time(e_end))
    build_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b, _ in marks) / args.steps)
    look_ms = max_over_ranks(sum(b.elapsed_time(c) for _, b, c in marks) / args.steps)
    ms = total_ms / args.steps
    # correctness of the last step against the generator's ground truth
    ok = bool(torch.equal(of, ef)) and bool(torch.equal(ov, ev))
    okt = torch.tensor([1 if ok else 0], device=dev)
    if world > 1:
        tdist.all_reduce(okt, op=tdist.ReduceOp.MIN)
    ok = bool(okt.item())

    # ---------------------------------------------------------------- roofline
    peak, peak_src = peaks()
    per_step = {k: v[1] / args.steps for k, v in kstats.items()}
    dom = max(per_step, key=per_step.get) if per_step else None
    roof = None
    if dom:
        launches_dom, ms_dom = kstats[dom]
        avg_ms = ms_dom / launches_dom
        # algorithmic bytes of each kernel: what it must move
        # per unit, with the table's actual S/n for the slot writes
        if dom.startswith("k_lookup"):
            units, bpu, what = n * args.steps / launches_dom, LOOKUP_BYTES_PER_QUERY, "queries"
        elif dom in ("k_partition", "k_split1", "k_split2"):
            units, bpu, what = n * args.steps / launches_dom, 32.0, "keys"  # read + write a 16-byte record
        else:  # k_bucket / k_split2_bucket: read the partition (16), write dir (8) + slots (16 S/n)
            units, bpu, what = n * args.steps / launches_dom, 16.0 + 8.0 + 16.0 * s_over_n, "keys"
        achieved = units * bpu / (avg_ms / 1e3) / 1e9
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
                summ = json.load(f)
            if dom in summ.get("kernels", {}):
                traffic = summ["kernels"][dom]["dram_bytes_per_launch"]
        except Exception:
            pass
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes": f"{bpu:.2f} B per {what[:-1]} x {int(units)} {what} per launch",
                "avg_launch_ms": round(avg_ms, 4), "share_of_step": round(per_step[dom] / ms, 4),
                "build_frac": round(n * BUILD_BYTES_PER_KEY / (build_ms / 1e3) / 1e9 / peak, 4),
                "lookup_frac": round(n * LOOKUP_BYTES_PER_QUERY / (look_ms / 1e3) / 1e9 / peak, 4)}

    # ---------------------------------------------------------------- e2e
    e2e = None
    if not args.no_e2e:
        hk = keys.cpu().pin_memory()
        hv = vals.cpu().pin_memory()
        hq = q.cpu().pin_memory()
        hov = torch.empty(n, dtype=torch.int64).pin_memory()
        hof = torch.empty(n, dtype=torch.uint8).pin_memory()

        def e2e_step():
            if not use_dist:
                m = hm.HashMap.build_u64(hk, hv, seed=0)  # host buffers: staged inside the C-ABI
                m.lookup(hq, hov, hof)  # host in, host out
                m.free()
            else:
                dk, dv, dq = hk.to(dev, non_blocking=True), hv.to(dev, non_blocking=True), hq.to(dev, non_blocking=True)
                m = hm.build_u64_dist(dk, dv, comm, seed=0, flags=dist_flags)
                v, f = hm.lookup_u64_dist(m, dq, comm)
                hov.copy_(v)
                hof.copy_(f)
                m.free()

        for _ in range(2):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        es = torch.cuda.Event(enable_timing=True)
        ee = torch.cuda.Event(enable_timing=True)
        es.record()
        ke = max(2, min(args.steps, 5))
        for _ in range(ke):
            e2e_step()
        ee.record()
        barrier()
        e2e_ms = max_over_ranks(max(es.elapsed_time(ee), 1e3 * (time.perf_counter() - t0)) / ke)
        e2e_ok = bool(torch.equal(hof, ef.cpu())) and bool(torch.equal(hov, ev.cpu()))
        e2e = {"value": round(n * world / (e2e_ms / 1e3) / 1e6, 2), "unit": "Mkeys/s",
               "h2d_bytes_per_step": 24 * n, "d2h_bytes_per_step": 9 * n, "ms_per_step": round(e2e_ms, 3),
               "correct": e2e_ok, "path": "hm_build_u64/hm_lookup_u64 on pinned host buffers" if not use_dist
               else "H2D copy + hm_build_u64_dist/hm_lookup_u64_dist + D2H copy"}
        del hk, hv, hq, hov, hof

    del keys, vals, q, ev, ef, ov, of
    torch.cuda.empty_cache()
    configs = None
    if not args.no_configs:
        configs = extra_configs(world, rank, dev, comm, peak, use_dist)

    if fused:
        hm.dist_release_windows(comm)  # (collective)
    if rank != 0:
        if use_dist:
            tdist.destroy_process_group()
        return 0
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline()
    out = {
        "metric": METRIC,
        "value": round(n * world / (ms / 1e3) / 1e6, 2),
        "unit": "Mkeys/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic: seeded splitmix64 key stream (workloads/gen.py, generated on device)",
        "config": dict(config_dict(world), **({"exchange": "fused route + NVLink window stores (HM_FLAG_FUSED_EXCHANGE)"}
                                              if fused else ({"exchange": fused_note or "route + grouped ncclSend/ncclRecv"}
                                                             if use_dist else {}))),
        "build_mkeys_s": round(n * world / (build_ms / 1e3) / 1e6, 2),
        "lookup_mq_s": round(n * world / (look_ms / 1e3) / 1e6, 2),
        "build_ms": round(build_ms, 4), "lookup_ms": round(look_ms, 4),
        "correct": ok,
        "roofline": roof,
        "kernels_ms_per_step": {k: round(v, 4) for k, v in sorted(per_step.items(), key=lambda x: -x[1])},
        "configs": configs,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if use_dist and world == 1:
        out["config"]["parallelism"] = "1 GPU through hm_build_u64_dist / hm_lookup_u64_dist (--dist-path)"
    print(json.dumps(out), flush=True)
    if use_dist:
        tdist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1/C3/C5 measurements after the timed region")
    ap.add_argument("--dist-path", action="store_true",
                    help="N = 1 through the sharded C calls on a one-rank NCCL group (checks the N > 1 code path)")
    ap.add_argument("--fused-exchange", action="store_true",
                    help="with --dist-path at N = 1: route straight into the NCCL window (HM_FLAG_FUSED_EXCHANGE, NEXT-2)")
    ap.add_argument("--no-fused-exchange", action="store_true",
                    help="N > 1: route + grouped ncclSend/ncclRecv instead of the fused route + window stores")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
