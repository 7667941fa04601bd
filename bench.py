"""Benchmark: doc pairs/s (and NW GCUPS) of the B200 miner hot path.

Default workload = BASELINE config 2: 10,000 synthetic doc pairs of 100 x 100
sentences per GPU (60 translation pairs + 40/40 one-sided distractors, 5k-word
dictionary, threshold 0.5, penalty 0.2). A step mines every document of the
batch: score -> NW -> traceback -> threshold -> record compaction (+ NCCL
gather of the records to rank 0 when N > 1).

  value  kernel-resident: packed inputs already in HBM, records left on device
  e2e    the same step through the C ABI with HOST buffers (bm_mine_host):
         pinned H2D of the packed batch, mining, D2H of the records
  cpu_baseline / --impl reference: the C restatement of the reference path
         (oracle/, "port") on the box's host cores, bounded sample

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
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


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_workload(n_docs: int, seed: int):
    from paper_1509_08639_b200 import synth

    return synth.make_corpus(*synth.c2_shape(n_docs), seed=seed)


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


# ----------------------------------------------------------------- CPU legs
def cpu_port_rate(sc, model, target_s: float, threads: int, max_docs: int):
    """Oracle mining throughput (doc pairs/s) on a bounded sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    oracle.build()
    plex = sc.world.packed_lexicon()
    c = sc.packed
    # calibrate on a small sample, then size the measured sample to ~target_s
    probe = min(64, c.n_docs)
    hb = oracle.HostBatch(c, plex, c.src0[:probe], c.n[:probe], c.tgt0[:probe], c.m[:probe])
    t0 = time.perf_counter()
    oracle.mine(hb, model, THRESHOLD, PENALTY, threads=threads)
    rate = probe / max(time.perf_counter() - t0, 1e-6)
    k = int(min(max_docs, max(probe, rate * target_s)))
    hb = oracle.HostBatch(c, plex, c.src0[:k], c.n[:k], c.tgt0[:k], c.m[:k])
    t0 = time.perf_counter()
    oracle.mine(hb, model, THRESHOLD, PENALTY, threads=threads)
    dt = time.perf_counter() - t0
    return k / dt, k, dt


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


def run_reference(args):
    """--impl reference: the CPU restatement of the reference path (oracle,
    kind "port": the reference itself is Python and has no compiled path)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1509_08639_b200.classifier import load_model

    model = load_model(MODEL)
    cores = host_cores()
    sc = make_workload(args.docs, seed=1)
    per_step = args.ref_docs
    rates = []
    for s in range(args.warmup + args.steps):
        # each step: a bounded sample of the workload (different docs each step)
        off = (s * per_step) % max(1, sc.packed.n_docs - per_step)
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle

        c = sc.packed
        sl = slice(off, off + per_step)
        hb = oracle.HostBatch(c, sc.world.packed_lexicon(), c.src0[sl], c.n[sl], c.tgt0[sl], c.m[sl])
        t0 = time.perf_counter()
        oracle.mine(hb, model, THRESHOLD, PENALTY, threads=cores)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            rates.append((per_step, dt))
    docs = sum(r[0] for r in rates)
    secs = sum(r[1] for r in rates)
    value = docs / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / len(rates),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{per_step} docs of the workload per step (100x100), "
                                   f"C restatement oracle/bimine_oracle.c, {cores} threads, "
                                   f"{cpu_model()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, world):
    return {
        "workload": "C2: synthetic doc pairs, 100x100 sentences (60 translation pairs + 40/40 "
                    "distractors), 5k-word dictionary, threshold 0.5, penalty 0.2",
        "docs_per_gpu": args.docs, "global_docs": args.docs * world,
        "cells_per_doc": 10000, "parallelism": f"dp{world}",
        "l2": "flushed between timed steps (256 MiB write)",
    }


# ----------------------------------------------------------------- GPU leg
def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1509_08639_b200 import _native as N
    from paper_1509_08639_b200 import engine, hostapi
    from paper_1509_08639_b200.classifier import load_model

    lib = N.lib()
    model = load_model(MODEL)
    t_gen = time.perf_counter()
    sc = make_workload(args.docs, seed=1 + rank)
    c = sc.packed
    plex = sc.world.packed_lexicon()
    log(f"[rank {rank}] workload: {c.n_docs} docs, {c.n_sent} sentences, "
        f"{c.tok_id.size} entries ({time.perf_counter() - t_gen:.1f}s)")

    dc = engine.DeviceCorpus.upload(c)
    dl = engine.DeviceLexicon.upload(plex)
    view = engine.DocView.of(c)
    n_h, m_h = view.n, view.m
    amax = np.ascontiguousarray(view.token_max(c), dtype=np.int32)
    dev = torch.device("cuda", local)
    rec_off = engine.record_offsets(n_h, m_h)
    cap = int(np.minimum(n_h, m_h).sum())
    rec = torch.empty(cap * 24, dtype=torch.uint8, device=dev)
    dense = torch.empty(cap * 24, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(c.n_docs, dtype=torch.int32, device=dev)
    cost = torch.empty(c.n_docs, dtype=torch.float64, device=dev)
    total = torch.zeros(1, dtype=torch.int64, device=dev)
    rec_off_d = engine.to_dev(rec_off, dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    sp = int(stream.cuda_stream)
    mstruct = N.model_struct(model)
    cells = int((n_h.astype(np.int64) * m_h).sum())

    def step():
        N.check(lib.bm_mine(C.byref(dc.sent), C.byref(view.docs), n_h.ctypes.data,
                            m_h.ctypes.data, amax.ctypes.data, C.byref(dl.lex), C.byref(mstruct),
                            THRESHOLD, PENALTY, engine._ptr(rec_off_d), engine._ptr(rec),
                            engine._ptr(cnt), engine._ptr(cost), sp))
        N.check(lib.bm_compact(engine._ptr(rec), engine._ptr(rec_off_d), engine._ptr(cnt),
                               c.n_docs, engine._ptr(dense), engine._ptr(total), sp))
        if world > 1:
            gather_records(dist, dense, total, rank, world, dev)

    def timed(fn, k, warm):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        times = []
        l0 = lib.bm_launches()
        for _ in range(k):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            times.append(a.elapsed_time(b))
        launches = lib.bm_launches() - l0
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return times, launches

    # clocks are sampled across every timed GPU region below (device-resident
    # steps, the dominant-kernel timing and the end-to-end steps)
    clk = ClockSampler(local).__enter__()
    times, launches = timed(step, args.steps, args.warmup)
    ms = float(np.mean(times))
    t_all = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_all, op=dist.ReduceOp.MAX)
    tot_ms = float(t_all.item())
    value = args.docs * world * args.steps / (tot_ms / 1e3)
    n_rec = int(total.item())

    # dominant-kernel timing on the launching stream (one fused launch = all docs)
    kern_ms = kernel_ms(lib, dc, view, dl, mstruct, n_h, m_h, amax, rec_off_d, rec, cnt, cost,
                        sp, stream, flush)
    peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    in_bytes = int(sum(getattr(c, k).nbytes for k in (
        "n_tok", "n_punct", "n_alpha", "tok_off", "tok_id", "tok_alpha", "dig_off", "dig_id")))
    alg_bytes = 8 * cells + in_bytes + 24 * n_rec
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    traffic, traffic_src, compute_util = measured_traffic()
    fp64 = fp64_roof(lib, torch, dev, stream)

    # end to end through the C ABI with host buffers (pinned)
    pb = hostapi.PinnedBatch(c, plex, pin=True)
    d2h = [0]

    def e2e_step():
        _, k, dbytes = hostapi.mine_pinned(pb, model, THRESHOLD, PENALTY, sp)
        d2h[0] = dbytes

    e_times, e_launch = timed(e2e_step, args.steps, max(1, args.warmup // 2))
    clk.__exit__(None, None, None)
    e_tot = torch.tensor([sum(e_times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e_tot, op=dist.ReduceOp.MAX)
    e2e_value = args.docs * world * args.steps / (float(e_tot.item()) / 1e3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:  # CPU baseline: N=1 only
        rate, k, dt = cpu_port_rate(sc, model, args.cpu_seconds, host_cores(), args.docs)
        cpu = {"value": rate, "unit": UNIT, "cores": host_cores(), "kind": "port",
               "sample": f"{k} docs of the workload (100x100) in {dt:.1f}s, oracle/bimine_oracle.c "
                         f"(C restatement of the reference path), {host_cores()} threads, "
                         f"{cpu_model()}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": workload_config(args, world),
            "nw_gcups": cells * world * args.steps / (tot_ms / 1e3) / 1e9,
            "records_per_step": n_rec,
            "roofline": {
                "bound": "hbm", "kernel": "bm_mine = hits_kernel + mine_ring_kernel<4>",
                "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic,
                "traffic_source": traffic_src,
                "alg_bytes_per_launch": alg_bytes,
                "alg_bytes_def": "SURVEY 8(d): 8 B/cell similarity matrix + packed inputs + records",
                "kernel_ms": kern_ms, "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst)",
            },
            "fp64": fp64,
            "compute_utilisation": compute_util,
            "clocks": clk.summary(),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": pb.h2d_bytes,
                    "d2h_bytes_per_step": d2h[0],
                    "path": "bm_mine_host: pinned host buffers -> H2D -> mine -> compact -> D2H"},
            "gpu_launches": int(launches),
            "gpu_launches_e2e": int(e_launch),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def kernel_ms(lib, dc, view, dl, mstruct, n_h, m_h, amax, rec_off_d, rec, cnt, cost, sp, stream,
              flush, reps: int = 5):
    """Average duration of one bm_mine launch set (fused kernel dominates)."""
    import torch

    from paper_1509_08639_b200 import _native as N
    from paper_1509_08639_b200 import engine

    out = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        N.check(lib.bm_mine(C.byref(dc.sent), C.byref(view.docs), n_h.ctypes.data,
                            m_h.ctypes.data, amax.ctypes.data, C.byref(dl.lex), C.byref(mstruct),
                            THRESHOLD, PENALTY, engine._ptr(rec_off_d), engine._ptr(rec),
                            engine._ptr(cnt), engine._ptr(cost), sp))
        b.record(stream)
        b.synchronize()
        out.append(a.elapsed_time(b))
    return float(np.mean(out[1:])) if len(out) > 1 else float(out[0])


def measured_traffic():
    """DRAM bytes of one C2 bm_mine launch pair from the committed ncu capture
    (profiles/, dram__bytes_read.sum + dram__bytes_write.sum), and the ring
    kernel's measured issue / FP64-pipe utilisation from the same capture."""
    pdir = os.path.join(ROOT, "profiles")
    prof = sorted(p for p in os.listdir(pdir) if p.endswith("_ncu_raw_metrics.json")) \
        if os.path.isdir(pdir) else []
    for name in reversed(prof):
        d = json.load(open(os.path.join(pdir, name)))
        if not all(k in d for k in ("hits_kernel", "mine_ring_kernel<4>")):
            continue
        tot = 0.0
        for k in ("hits_kernel", "mine_ring_kernel<4>"):
            tot += float(d[k]["dram__bytes_read.sum"]) + float(d[k]["dram__bytes_write.sum"])
        ring = d["mine_ring_kernel<4>"]
        util = {
            "kernel": "mine_ring_kernel<4>",
            "issue_slots_busy_pct": ring.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "fp64_pipe_active_pct": ring.get(
                "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "stall_share": ring.get("stall_share"),
            "source": f"profiles/{name}",
        }
        return tot * 1e6, f"profiles/{name} (ncu --set full, MB -> bytes)", util
    return None, None, None


def fp64_roof(lib, torch, dev, stream):
    """Measured FP64 FMA throughput of the device (8 DFMA chains / thread)."""
    from paper_1509_08639_b200 import _native as N

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    blocks, iters = sms * 8, 4096
    sp = int(stream.cuda_stream)
    N.check(lib.bm_probe_fp64(out.data_ptr(), iters, blocks, sp))
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    N.check(lib.bm_probe_fp64(out.data_ptr(), iters, blocks, sp))
    b.record(stream)
    b.synchronize()
    ms = a.elapsed_time(b)
    flops = 2.0 * 8 * 256 * blocks * iters
    return {"dfma_tflops": flops / (ms / 1e3) / 1e12, "probe": "8 independent DFMA chains x 256 thr"}


def gather_records(dist, dense, total, rank, world, dev):
    """Rank 0 receives every rank's compacted records over NCCL (the only
    collective of the path): sizes first, then the padded record buffers."""
    import torch

    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, total)
    mx = int(max(int(s.item()) for s in sizes))
    buf = dense[: mx * 24] if mx > 0 else dense[:24]
    if rank == 0:
        outs = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, outs, dst=0)
    else:
        dist.gather(buf, None, dst=0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--docs", type=int, default=10000)
    ap.add_argument("--ref-docs", type=int, default=2000)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
