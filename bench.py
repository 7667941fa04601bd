"""Benchmark: doc pairs/s (and NW GCUPS) of the B200 miner hot path.

Workloads (BASELINE.json configs; --workload, default c3):

  c3  1,000,000 synthetic doc pairs with skewed lengths (n = LogNormal(ln 60, 1)
      clipped to 10..2000 sentences, m = n * LogNormal(0, 0.25)), the config
      quoted "across 8 x B200": at N GPUs the ONE global corpus is split by
      LPT over n*m (shard.lpt_shards), every rank mines its shard, the
      compacted records are gathered to rank 0 over NCCL and put back in
      global document order on the device (bm_merge_shards). scaling: strong.
  c2  10,000 doc pairs of 100 x 100 sentences per GPU (scaling: weak).
  c4  one 8192 x 8192 pair, scored, aligned and extracted (replicas at N > 1).
  c5  tuning sweep: 100,000 doc pairs (C2-shaped) x 8 penalties x 8 thresholds.

A step mines every document of the workload once: score -> NW -> traceback ->
threshold -> record compaction (c5: score once, one DP per penalty, counts per
grid point). Inputs are synthetic, generated per document by the native
generator (csrc/bm_synth.cpp, the reference test generator's distributions).

  value  kernel-resident: packed inputs already in HBM, records on the device
  e2e    the same step through the C ABI with HOST buffers (bm_mine_host_*):
         pinned H2D of the packed batch, mining, D2H of the records
  cpu_baseline / --impl reference: the C restatement of the reference path
         (oracle/, "port") on the box's host cores, bounded sample

At N = 1 the default run also measures c2, c4 and c5 ("workloads") so every
BASELINE config is timed by the driver, with clocks.

Usage: python bench.py [--workload c3|c2|c4|c5] [--gpus N] [--steps K] [--warmup W]
                       [--impl ours|reference]
       torchrun --nproc-per-node N bench.py --gpus N ...
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MODEL = os.path.join(ROOT, "tests", "golden", "model5k_fwd.json")
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
THRESHOLD, PENALTY = 0.5, 0.2
METRIC = "doc pairs/sec and NW GCUPS at 1/2/4/8 B200 vs CPU reference"
UNIT = "doc pairs/s"
C3_DOCS, C3_SEED = 1_000_000, 2026
C5_PENS = [0.05, 0.1, 0.2, 0.3, 0.4, 0.6, 0.8, 1.6]
C5_THRS = [0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9]
DP_OPS_PER_CELL = 7  # 1-S, diag add, one shared +p, two min, two code compares


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampled every 100 ms while the timed regions run (entering
    waits for the first sample, so the sampler is live before timing starts)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", os.environ.get("BM_CLOCK_MS", "100")],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- inputs
def c3_shapes(n_docs: int):
    from paper_1509_08639_b200 import synth

    return synth.c3_shape(n_docs, seed=C3_SEED)


def gen_docs(g, a, b, ids, seed):
    from paper_1509_08639_b200 import synth

    return synth.make_corpus_native(g, a, b, ids=ids, seed=seed)


def workload_spec(name: str, args, world: int) -> dict:
    if name == "c3":
        return {"workload": f"C3: {args.c3_docs} synthetic doc pairs, skewed lengths "
                            "(n = LogNormal(ln 60, 1) clipped to 10..2000, m = n * LogNormal(0, 0.25)), "
                            "60% translation pairs, 5k-word dictionary, threshold 0.5, penalty 0.2",
                "global_docs": args.c3_docs, "docs_per_gpu": None,
                "parallelism": f"dp{world} (LPT shards of one corpus, NCCL gather to rank 0)",
                "scaling": "strong"}
    if name == "c2":
        return {"workload": "C2: synthetic doc pairs, 100x100 sentences (60 translation pairs + "
                            "40/40 distractors), 5k-word dictionary, threshold 0.5, penalty 0.2",
                "global_docs": args.c2_docs * world, "docs_per_gpu": args.c2_docs,
                "parallelism": f"dp{world} (independent batches)", "scaling": "weak"}
    if name == "c4":
        return {"workload": "C4: one 8192x8192 synthetic doc pair (4915 translation pairs + "
                            "3277/3277 distractors), scored, aligned, extracted; threshold 0.5, "
                            "penalty 0.2", "global_docs": world, "docs_per_gpu": 1,
                "parallelism": f"replicas x{world}", "scaling": "weak"}
    if name == "c5":
        return {"workload": f"C5: tuning sweep, {args.c5_docs} doc pairs of 100x100 x "
                            f"{len(C5_PENS)} penalties x {len(C5_THRS)} thresholds "
                            "(score once, one DP per penalty, pred/gold-hit counts per grid point)",
                "global_docs": args.c5_docs * world, "docs_per_gpu": args.c5_docs,
                "parallelism": f"dp{world} (independent dev sets)", "scaling": "weak"}
    raise ValueError(name)


def local_docs(name: str, args, rank: int, world: int):
    """(g, a, b, global ids, seed) of this rank's documents."""
    if name == "c3":
        from paper_1509_08639_b200 import shard

        g, a, b = c3_shapes(args.c3_docs)
        idx = shard.lpt_shards(g + a, g + b, world)[rank]
        return g[idx], a[idx], b[idx], idx, C3_SEED
    if name == "c2":
        k = args.c2_docs
        return (np.full(k, 60), np.full(k, 40), np.full(k, 40),
                np.arange(rank * k, (rank + 1) * k), 1)
    if name == "c4":
        return np.array([4915]), np.array([3277]), np.array([3277]), np.array([rank]), 404
    if name == "c5":
        k = args.c5_docs
        return (np.full(k, 60), np.full(k, 40), np.full(k, 40),
                np.arange(rank * k, (rank + 1) * k), 55)
    raise ValueError(name)


# ----------------------------------------------------------------- CPU legs
def oracle_mod():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle  # checker / CPU baseline only

    oracle.build()
    return oracle


def oracle_step(oracle, name, model, sc, threads):
    """One oracle pass over a generated sample (NativeSynthCorpus)."""
    plex = sc.world.packed_lexicon()
    hb = oracle.HostBatch(sc.packed, plex)
    if name == "c5":
        keys = sc.gold_keys()
        oracle.tune(hb, model, C5_PENS, C5_THRS, keys, threads=threads)
    else:
        oracle.mine(hb, model, THRESHOLD, PENALTY, threads=threads)


def sample_docs(name, args, k, seed):
    """k documents drawn uniformly from the workload (g, a, b, ids, seed)."""
    r = np.random.default_rng(seed)
    if name == "c3":
        g, a, b = c3_shapes(args.c3_docs)
        ids = np.sort(r.choice(args.c3_docs, size=min(k, args.c3_docs), replace=False))
        return g[ids], a[ids], b[ids], ids, C3_SEED
    if name == "c4":
        return np.array([4915]), np.array([3277]), np.array([3277]), np.array([0]), 404
    total = args.c2_docs if name == "c2" else args.c5_docs
    ids = np.sort(r.choice(total, size=min(k, total), replace=False))
    s = 1 if name == "c2" else 55
    return np.full(ids.size, 60), np.full(ids.size, 40), np.full(ids.size, 40), ids, s


def cpu_rate(name, args, model, target_s: float, threads: int, seed: int = 99):
    """Oracle throughput (doc pairs/s) on a bounded uniform sample of the
    workload, sized by a calibration pass to about target_s seconds."""
    oracle = oracle_mod()
    probe = 1 if name == "c4" else 64
    sc = gen_docs(*sample_docs(name, args, probe, seed))
    t0 = time.perf_counter()
    oracle_step(oracle, name, model, sc, threads)
    dt = max(time.perf_counter() - t0, 1e-6)
    if name == "c4":
        return 1.0 / dt, 1, dt
    k = int(max(probe, min(args.ref_docs_max, probe / dt * target_s)))
    sc = gen_docs(*sample_docs(name, args, k, seed + 1))
    k = sc.packed.n_docs  # the sample never exceeds the workload
    t0 = time.perf_counter()
    oracle_step(oracle, name, model, sc, threads)
    dt = time.perf_counter() - t0
    return k / dt, k, dt


def run_reference(args):
    """--impl reference: the CPU restatement of the reference path (oracle,
    kind "port": the reference itself is Python + numba and has no compiled
    library to build), all host threads, a bounded sample per step."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1509_08639_b200.classifier import load_model

    model = load_model(MODEL)
    oracle = oracle_mod()
    cores = host_cores()
    name = args.workload
    # size one step to ~args.ref_step_s of oracle work
    sc = gen_docs(*sample_docs(name, args, 1 if name == "c4" else 64, 7))
    t0 = time.perf_counter()
    oracle_step(oracle, name, model, sc, cores)
    per_doc = max(time.perf_counter() - t0, 1e-6) / max(sc.packed.n_docs, 1)
    k = 1 if name == "c4" else int(max(64, min(args.ref_docs_max, args.ref_step_s / per_doc)))
    rates = []
    for s in range(args.warmup + args.steps):
        sc = gen_docs(*sample_docs(name, args, k, 1000 + s))
        t0 = time.perf_counter()
        oracle_step(oracle, name, model, sc, cores)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            rates.append((sc.packed.n_docs, dt))
    docs = sum(r[0] for r in rates)
    secs = sum(r[1] for r in rates)
    value = docs / secs
    spec = workload_spec(name, args, world)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / len(rates),
        "higher_is_better": True, "scaling": spec["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": config_of(spec),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{k} docs drawn uniformly from the workload per step, "
                                   f"C restatement oracle/bimine_oracle.c, {cores} threads, "
                                   f"{cpu_model()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_of(spec: dict) -> dict:
    cfg = {k: v for k, v in spec.items() if k != "scaling" and v is not None}
    cfg["l2"] = "flushed between timed steps (256 MiB write)"
    return cfg


# ----------------------------------------------------------------- GPU leg
class Ctx:
    def __init__(self, args, rank, world, local):
        import torch

        from paper_1509_08639_b200 import _native as N
        from paper_1509_08639_b200.classifier import load_model

        self.args, self.rank, self.world, self.local = args, rank, world, local
        self.torch = torch
        self.N = N
        self.lib = N.lib()
        self.dev = torch.device("cuda", local)
        self.stream = torch.cuda.current_stream()
        self.sp = int(self.stream.cuda_stream)
        self.model = load_model(MODEL)
        self.mstruct = N.model_struct(self.model)
        self.flush = torch.empty(256 << 20, dtype=torch.uint8, device=self.dev)

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier()

    def timed(self, fn, k, warm):
        torch = self.torch
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        self.barrier()
        torch.cuda.synchronize()
        times = []
        l0 = self.lib.bm_launches()
        for _ in range(k):
            self.flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(self.stream)
            fn()
            b.record(self.stream)
            b.synchronize()
            times.append(a.elapsed_time(b))
        launches = self.lib.bm_launches() - l0
        torch.cuda.synchronize()
        self.barrier()
        return times, launches

    def max_over_ranks(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch.distributed as dist

        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())


class MineWorkload:
    """c2 / c3 / c4: bm_mine + bm_compact over the rank's documents."""

    def __init__(self, ctx: Ctx, name: str):
        from paper_1509_08639_b200 import engine

        self.ctx, self.name = ctx, name
        torch = ctx.torch
        t0 = time.perf_counter()
        g, a, b, ids, seed = local_docs(name, ctx.args, ctx.rank, ctx.world)
        self.ids = np.asarray(ids, dtype=np.int64)
        self.sc = gen_docs(g, a, b, ids, seed)
        c = self.c = self.sc.packed
        self.plex = self.sc.world.packed_lexicon()
        t1 = time.perf_counter()
        self.dc = engine.DeviceCorpus.upload(c)
        self.dl = engine.DeviceLexicon.upload(self.plex)
        self.view = engine.DocView.of(c)
        self.n_h = np.ascontiguousarray(c.n, np.int32)
        self.m_h = np.ascontiguousarray(c.m, np.int32)
        self.amax = np.ascontiguousarray(self.dc.doc_token_max(self.view), np.int32)
        self.rec_off_d = engine.to_dev(engine.record_offsets(self.n_h, self.m_h), ctx.dev)
        cap = int(np.minimum(self.n_h, self.m_h).clip(min=0).sum())
        self.rec = torch.empty(max(cap, 1) * 24, dtype=torch.uint8, device=ctx.dev)
        self.dense = torch.empty(max(cap, 1) * 24, dtype=torch.uint8, device=ctx.dev)
        self.cnt = torch.zeros(max(c.n_docs, 1), dtype=torch.int32, device=ctx.dev)
        self.cost = torch.empty(max(c.n_docs, 1), dtype=torch.float64, device=ctx.dev)
        self.total = torch.zeros(1, dtype=torch.int64, device=ctx.dev)
        self.cells = int((self.n_h.astype(np.int64) * self.m_h).sum())
        self.ids_d = engine.to_dev(self.ids.astype(np.int32), ctx.dev)
        self.gather = Gather(ctx, self.global_docs()) if (name == "c3" and ctx.world > 1) else None
        log(f"[rank {ctx.rank}] {name}: {c.n_docs} docs, {c.n_sent} sentences, {c.tok_id.size} "
            f"entries, {self.cells} cells (generated {t1 - t0:.1f}s, uploaded "
            f"{time.perf_counter() - t1:.1f}s)")

    def global_docs(self) -> int:
        return self.ctx.args.c3_docs if self.name == "c3" else self.c.n_docs * self.ctx.world

    def mine(self):
        from paper_1509_08639_b200 import engine

        ctx = self.ctx
        ctx.N.check(ctx.lib.bm_mine(C.byref(self.dc.sent), C.byref(self.view.docs),
                                    self.n_h.ctypes.data, self.m_h.ctypes.data,
                                    self.amax.ctypes.data, C.byref(self.dl.lex),
                                    C.byref(ctx.mstruct), THRESHOLD, PENALTY,
                                    engine._ptr(self.rec_off_d), engine._ptr(self.rec),
                                    engine._ptr(self.cnt), engine._ptr(self.cost), ctx.sp))

    def step(self):
        from paper_1509_08639_b200 import engine

        ctx = self.ctx
        self.mine()
        ctx.N.check(ctx.lib.bm_compact(engine._ptr(self.rec), engine._ptr(self.rec_off_d),
                                       engine._ptr(self.cnt), self.c.n_docs,
                                       engine._ptr(self.dense), engine._ptr(self.total), ctx.sp))
        if self.gather is not None:
            self.gather.run(self.dense, self.total, self.ids_d)

    # end to end: host buffers through the C ABI
    def e2e_setup(self):
        from paper_1509_08639_b200 import hostapi

        t0 = time.perf_counter()
        self.pb = hostapi.PinnedBatch(self.c, self.plex, pin=True)
        log(f"[rank {self.ctx.rank}] {self.name}: pinned {self.pb.fmt} host batch "
            f"{self.pb.h2d_bytes / 1e9:.2f} GB ({time.perf_counter() - t0:.1f}s)")
        self.d2h = 0
        self.h2d_extra = 0

    def e2e_step(self):
        from paper_1509_08639_b200 import hostapi

        ctx = self.ctx
        recs, k, d2h = hostapi.mine_pinned(self.pb, ctx.model, THRESHOLD, PENALTY, ctx.sp)
        self.d2h = d2h
        if self.gather is not None:
            # the rank's host records go to rank 0 over NCCL (H2D, gather,
            # order restore on the device, D2H of the merged records on rank 0)
            torch = ctx.torch
            raw = torch.from_numpy(recs.view(np.uint8).reshape(-1))
            dbuf = raw.to(ctx.dev, non_blocking=True)
            tot = torch.tensor([k], dtype=torch.int64, device=ctx.dev)
            self.h2d_extra = k * 24
            merged = self.gather.run(dbuf, tot, self.ids_d)
            if merged is not None:
                host = torch.empty(merged.numel(), dtype=torch.uint8, pin_memory=True)
                host.copy_(merged)
                self.d2h = int(merged.numel())

    def e2e_bytes(self):
        return self.pb.h2d_bytes + self.h2d_extra, self.d2h

    def alg_bytes(self, n_rec: int) -> int:
        c = self.c
        in_bytes = int(sum(getattr(c, k).nbytes for k in (
            "n_tok", "n_punct", "n_alpha", "tok_off", "tok_id", "tok_alpha", "dig_off", "dig_id")))
        return 8 * self.cells + in_bytes + 24 * n_rec

    def kernel_ms(self, reps=3):
        """Average duration of one bm_mine launch set (CUDA events on its stream)."""
        torch = self.ctx.torch
        out = []
        for _ in range(reps + 1):
            self.ctx.flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(self.ctx.stream)
            self.mine()
            b.record(self.ctx.stream)
            b.synchronize()
            out.append(a.elapsed_time(b))
        return float(np.mean(out[1:]))


class Gather:
    """Rank r's compacted records (local document indices) -> rank 0, in global
    document order: ids remap on each rank, an all_gather of record counts, an
    NCCL gather of padded 24-byte record buffers, bm_merge_shards on rank 0."""

    def __init__(self, ctx: Ctx, n_docs: int):
        self.ctx, self.n_docs = ctx, n_docs
        torch = ctx.torch
        self.out = None
        self.total = torch.zeros(1, dtype=torch.int64, device=ctx.dev)

    def run(self, dense, total, ids_d):
        import torch.distributed as dist

        from paper_1509_08639_b200 import engine

        ctx = self.ctx
        torch = ctx.torch
        counts = [torch.zeros(1, dtype=torch.int64, device=ctx.dev) for _ in range(ctx.world)]
        dist.all_gather(counts, total)
        sizes = torch.cat(counts)
        mx = max(int(sizes.max().item()), 1)
        k = int(total.item())
        recs = dense[: k * 24].view(torch.int32).view(-1, 6)
        buf = torch.zeros((mx, 6), dtype=torch.int32, device=ctx.dev)
        if k:
            buf[:k] = recs
            buf[:k, 0] = ids_d[recs[:, 0].long()]  # local -> global document index
        if ctx.rank == 0:
            parts = torch.empty((ctx.world, mx, 6), dtype=torch.int32, device=ctx.dev)
            dist.gather(buf, list(parts.unbind(0)), dst=0)
            if self.out is None or self.out.numel() < ctx.world * mx * 24:
                self.out = torch.empty(ctx.world * mx * 24, dtype=torch.uint8, device=ctx.dev)
            ctx.N.check(ctx.lib.bm_merge_shards(engine._ptr(parts), mx, engine._ptr(sizes),
                                                ctx.world, self.n_docs, engine._ptr(self.out),
                                                engine._ptr(self.total), ctx.sp))
            return self.out[: int(sizes.sum().item()) * 24]
        dist.gather(buf, None, dst=0)
        return None


class TuneWorkload:
    """c5: bm_tune over the rank's dev set (device-resident gold keys)."""

    def __init__(self, ctx: Ctx, name: str):
        from paper_1509_08639_b200 import engine

        self.ctx, self.name = ctx, name
        t0 = time.perf_counter()
        g, a, b, ids, seed = local_docs(name, ctx.args, ctx.rank, ctx.world)
        self.sc = gen_docs(g, a, b, ids, seed)
        c = self.c = self.sc.packed
        self.plex = self.sc.world.packed_lexicon()
        self.keys = self.sc.gold_keys()
        self.gk, self.goff = engine.pack_gold(self.keys)
        t1 = time.perf_counter()
        self.dc = engine.DeviceCorpus.upload(c)
        self.dl = engine.DeviceLexicon.upload(self.plex)
        self.view = engine.DocView.of(c)
        self.gold = engine.DeviceGold(self.gk, self.goff)
        self.cells = int((c.n.astype(np.int64) * c.m).sum())
        log(f"[rank {ctx.rank}] c5: {c.n_docs} docs, {self.cells} cells, "
            f"{self.gk.size} gold keys (generated {t1 - t0:.1f}s)")

    def global_docs(self) -> int:
        return self.c.n_docs * self.ctx.world

    def step(self):
        from paper_1509_08639_b200 import engine

        engine.tune_counts_device(self.dc, self.dl, self.view, self.ctx.model, C5_PENS, C5_THRS,
                                  self.gold)

    def kernel_ms(self, reps=3):
        torch = self.ctx.torch
        out = []
        for _ in range(reps + 1):
            self.ctx.flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(self.ctx.stream)
            self.step()
            b.record(self.ctx.stream)
            b.synchronize()
            out.append(a.elapsed_time(b))
        return float(np.mean(out[1:]))

    def e2e_setup(self):
        from paper_1509_08639_b200 import hostapi

        self.tp = hostapi.TunePinned(self.c, self.gk, self.goff)
        self.h2d = self.tp.h2d_bytes
        self.d2h = 2 * len(C5_PENS) * len(C5_THRS) * 8

    def e2e_step(self):
        """Page-locked host dev set -> device, chunk by chunk, each chunk's copy
        overlapping the previous chunk's bm_tune (hostapi.tune_pinned) -> counts
        to the host -> precision/recall/F1 of every grid point
        (tuner.py:67-84, 134-147)."""
        from paper_1509_08639_b200 import hostapi, tuner

        p, h = hostapi.tune_pinned(self.tp, self.dl, self.ctx.model, C5_PENS, C5_THRS)
        n_gold = int(self.gk.size)
        trace = [tuner._prf(int(p[a, b]), n_gold, int(h[a, b]))
                 for b in range(len(C5_THRS)) for a in range(len(C5_PENS))]
        self.best = max(trace)

    def e2e_bytes(self):
        return self.h2d, self.d2h

    def alg_bytes(self, n_rec: int) -> int:
        c = self.c
        in_bytes = int(sum(getattr(c, k).nbytes for k in (
            "n_tok", "n_punct", "n_alpha", "tok_off", "tok_id", "tok_alpha", "dig_off", "dig_id")))
        return 8 * self.cells + in_bytes


def measured_profile(name: str, cells: int):
    """DRAM bytes (scaled to `cells` from the capture's profiled cells) and
    issue / FP64-pipe utilisation of the workload's kernels from the latest
    committed ncu --set full capture (profiles/*_<name>_ncu_raw_metrics.json)."""
    pdir = os.path.join(ROOT, "profiles")
    if not os.path.isdir(pdir):
        return None
    cands = sorted(p for p in os.listdir(pdir) if p.endswith(f"_{name}_ncu_raw_metrics.json"))
    if not cands:
        return None
    d = json.load(open(os.path.join(pdir, cands[-1])))
    kernels = {k: v for k, v in d.items() if isinstance(v, dict) and "dram__bytes_read.sum" in v}
    if not kernels:
        return None
    traffic = sum(float(v["dram__bytes_read.sum"]) + float(v["dram__bytes_write.sum"])
                  for v in kernels.values()) * float(d.get("bytes_scale", 1e6))
    if d.get("profiled_cells"):
        traffic *= cells / float(d["profiled_cells"])
    top = max(kernels.items(), key=lambda kv: float(kv[1].get("gpu__time_duration.sum", 0)))
    return {"traffic": traffic, "source": f"profiles/{cands[-1]}",
            "traffic_per_cell": traffic / max(cells, 1),
            "top_kernel": top[0],
            "issue_slots_busy_pct": top[1].get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "fp64_pipe_active_pct": top[1].get(
                "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "per_launch_scale": d.get("per_launch_scale", 1.0)}


def fp64_roof(ctx: Ctx):
    """Measured FP64 FMA throughput of the device (8 DFMA chains / thread)."""
    torch = ctx.torch
    sms = torch.cuda.get_device_properties(ctx.dev).multi_processor_count
    out = torch.zeros(1, dtype=torch.float64, device=ctx.dev)
    blocks, iters = sms * 8, 4096
    ctx.N.check(ctx.lib.bm_probe_fp64(out.data_ptr(), iters, blocks, ctx.sp))
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(ctx.stream)
    ctx.N.check(ctx.lib.bm_probe_fp64(out.data_ptr(), iters, blocks, ctx.sp))
    b.record(ctx.stream)
    b.synchronize()
    ms = a.elapsed_time(b)
    flops = 2.0 * 8 * 256 * blocks * iters
    return {"dfma_tflops": flops / (ms / 1e3) / 1e12, "probe": "8 independent DFMA chains x 256 thr"}


def measure(ctx: Ctx, name: str, steps: int, warmup: int, cpu: bool, fp64: dict):
    """Device-resident steps, the dominant launch set, end-to-end steps and
    (rank 0, N = 1) the CPU baseline of one workload -> the line's fields."""
    args = ctx.args
    w = TuneWorkload(ctx, name) if name == "c5" else MineWorkload(ctx, name)
    times, launches = ctx.timed(w.step, steps, warmup)
    tot_ms = ctx.max_over_ranks(sum(times))
    gdocs = w.global_docs()
    value = gdocs * steps / (tot_ms / 1e3)
    n_rec = int(w.total.item()) if hasattr(w, "total") else 0
    kern_ms = ctx.max_over_ranks(w.kernel_ms())
    peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    alg = w.alg_bytes(n_rec)
    achieved = alg / (kern_ms / 1e3) / 1e9
    prof = measured_profile(name, w.cells)
    npen = len(C5_PENS) if name == "c5" else 1
    dp_cells_s = w.cells * npen / (kern_ms / 1e3)
    dp_peak_cells = fp64["dfma_tflops"] * 1e12 / 2 / DP_OPS_PER_CELL
    kernel_set = ("bm_tune = score (hits_doc + score_hits) + nw_band<4 penalties> + tune_count"
                  if name == "c5" else "bm_mine = hits + mine_ring (fused tier) + banded tier")
    roof = {"bound": "hbm", "kernel": kernel_set, "achieved": achieved, "peak": hbm_peak,
            "unit": "GB/s", "frac": achieved / hbm_peak,
            "traffic": None if prof is None else prof["traffic"],
            "alg_bytes_per_launch": alg,
            "alg_bytes_def": "SURVEY 8(d): 8 B/cell similarity matrix + packed inputs + 24 B/record",
            "kernel_ms": kern_ms, "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst)"}
    if prof is not None:
        roof["traffic_source"] = prof["source"] + " (DRAM bytes per cell of the capture x this step's cells)"
        roof["traffic_bytes_per_cell"] = prof["traffic_per_cell"]
        roof["measured_dram_gbs"] = prof["traffic"] / (kern_ms / 1e3) / 1e9
        roof["measured_dram_frac"] = roof["measured_dram_gbs"] / hbm_peak
    dp = {"achieved_gcups": dp_cells_s / 1e9, "peak_gcups": dp_peak_cells / 1e9,
          "frac": dp_cells_s / dp_peak_cells,
          "def": f"DP cells x {DP_OPS_PER_CELL} FP64 ops / (measured DFMA rate / 2 flops)",
          "penalties_per_cell": npen}
    if prof is not None:
        dp["issue_slots_busy_pct"] = prof["issue_slots_busy_pct"]
        dp["fp64_pipe_active_pct"] = prof["fp64_pipe_active_pct"]
        dp["top_kernel"] = prof["top_kernel"]
    w.e2e_setup()
    e_times, e_launch = ctx.timed(w.e2e_step, steps, max(1, warmup // 2))
    e_tot = ctx.max_over_ranks(sum(e_times))
    h2d, d2h = w.e2e_bytes()
    res = {
        "value": value, "ms_per_step": float(np.mean(times)), "steps": steps, "warmup": warmup,
        "nw_gcups": global_cells(ctx, w) * npen * steps / (tot_ms / 1e3) / 1e9,
        "records_per_step": n_rec, "roofline": roof, "roofline_dp_alu": dp,
        "e2e": {"value": gdocs * steps / (e_tot / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "path": ("hostapi.tune_pinned: page-locked dev set -> chunked H2D overlapping "
                         "bm_tune per chunk -> counts D2H -> P/R/F1"
                         if name == "c5" else
                         "bm_mine_host_*: pinned host buffers -> H2D -> mine -> compact -> D2H"
                         + (" -> NCCL gather -> bm_merge_shards on rank 0" if ctx.world > 1
                            and name == "c3" else ""))},
        "gpu_launches": int(launches), "gpu_launches_e2e": int(e_launch),
        "cells_per_step": w.cells,
    }
    if cpu and ctx.rank == 0 and ctx.world == 1 and not args.no_cpu:
        rate, k, dt = cpu_rate(name, args, ctx.model, args.cpu_seconds, host_cores())
        res["cpu_baseline"] = {
            "value": rate, "unit": UNIT, "cores": host_cores(), "kind": "port",
            "sample": f"{k} docs drawn uniformly from the workload, {dt:.1f}s, oracle/bimine_oracle.c "
                      f"(C restatement of the reference path), {host_cores()} threads, {cpu_model()}"}
    del w
    ctx.torch.cuda.synchronize()
    ctx.lib.bm_trim()  # the next workload starts from an empty scratch
    ctx.torch.cuda.empty_cache()
    return res


def global_cells(ctx: Ctx, w) -> int:
    if ctx.world == 1:
        return w.cells
    import torch.distributed as dist

    t = ctx.torch.tensor([w.cells], dtype=ctx.torch.int64, device=ctx.dev)
    dist.all_reduce(t)
    return int(t.item())


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = Ctx(args, rank, world, local)
    # clocks are sampled across every timed GPU region below
    clk = ClockSampler(local).__enter__()
    fp64 = fp64_roof(ctx)
    main = measure(ctx, args.workload, args.steps, args.warmup, cpu=True, fp64=fp64)
    extras = {}
    todo = [] if args.extras in ("", "none") else args.extras.split(",")
    if world == 1:
        for name in todo:
            if name == args.workload:
                continue
            ks = max(3, args.steps // 2)
            extras[name] = measure(ctx, name, ks, max(3, args.warmup), cpu=not args.no_cpu_extras,
                                   fp64=fp64)
            extras[name]["config"] = config_of(workload_spec(name, args, world))
    clk.__exit__(None, None, None)
    if rank == 0:
        spec = workload_spec(args.workload, args, world)
        line = {
            "metric": METRIC, "value": main["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": main["ms_per_step"],
            "higher_is_better": True, "scaling": spec["scaling"], "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (native per-document generator, reference "
                                    "synthgen distributions)",
            "config": config_of(spec),
            "nw_gcups": main["nw_gcups"],
            "records_per_step": main["records_per_step"],
            "roofline": main["roofline"],
            "roofline_dp_alu": main["roofline_dp_alu"],
            "fp64": fp64,
            "clocks": clk.summary(),
            "e2e": main["e2e"],
            "gpu_launches": main["gpu_launches"],
            "gpu_launches_e2e": main["gpu_launches_e2e"],
            "cpu_baseline": main.get("cpu_baseline"),
        }
        if extras:
            line["workloads"] = extras
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=("c2", "c3", "c4", "c5"), default="c3")
    ap.add_argument("--extras", default="c2,c4,c5",
                    help="other workloads measured in the same run at N = 1 ('none' to skip)")
    ap.add_argument("--c3-docs", type=int, default=C3_DOCS)
    ap.add_argument("--c2-docs", type=int, default=10000)
    ap.add_argument("--c5-docs", type=int, default=100000)
    ap.add_argument("--ref-step-s", type=float, default=3.0)
    ap.add_argument("--ref-docs-max", type=int, default=200000)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cpu-extras", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
