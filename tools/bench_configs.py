"""Measure the non-headline BASELINE configs on one B200 (parity-checked):

  C1  one 200x200 document pair (5k dictionary), mine_corpus end to end
  C3  skewed corpus (n, m ~ LogNormal, 10..2000 sentences), both tiers
  C4  one 8192x8192 pair: DP-only GCUPS on the reference's random matrix
  C5  tuning sweep, 8 penalties x 8 thresholds, docs shaped like C2
  C5w the worst case of 64 distinct penalties x 1 threshold

Prints one JSON line per config. Usage: python tools/bench_configs.py [--c3-docs N] ...
"""

from __future__ import annotations

import argparse
import io
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (checker only)
import paper_1509_08639_b200 as bm  # noqa: E402
from paper_1509_08639_b200 import engine, synth  # noqa: E402

MODEL = os.path.join(ROOT, "tests", "golden", "model5k_fwd.json")


def cuda_ms(fn, reps=3):
    st = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        out.append(a.elapsed_time(b))
    return float(np.median(out))


def c1(model, lex):
    path = os.path.join(ROOT, "tests", "golden", "doc200.jsonl")
    doc = json.loads(open(path).read().strip())
    pair = bm.parse_document_pair(doc, "mem", 1)
    cfg = bm.MinerConfig(bm.MiningParams(0.5, 0.2))
    walls = []
    for _ in range(3):  # first call: one-time device init; then steady state
        t0 = time.perf_counter()
        sink = io.StringIO()
        bm.mine_corpus([pair], model, None, lex, cfg, sink)
        walls.append(time.perf_counter() - t0)
    ok = sink.getvalue() == open(os.path.join(ROOT, "tests", "golden", "mine200_fwd.tsv")).read()
    return {"config": "C1 200x200 single pair", "wall_ms_first_call": 1e3 * walls[0],
            "wall_ms_mine_corpus": 1e3 * min(walls[1:]), "tsv_identical_to_reference": ok}


def kernel_resident_ms(dc, dl, view, model, reps=3):
    """bm_mine + bm_compact with inputs and records resident on the device
    (SURVEY 8(d) "kernel-resident"); host planning inside bm_mine included."""
    import ctypes as C
    from paper_1509_08639_b200 import _native as N

    lib = N.lib()
    n_h, m_h = np.ascontiguousarray(view.n, np.int32), np.ascontiguousarray(view.m, np.int32)
    amax = np.ascontiguousarray(dc.doc_token_max(view), np.int32)
    dev = torch.device("cuda")
    rec_off = engine.record_offsets(n_h, m_h)
    cap = int(np.minimum(n_h, m_h).sum())
    rec = torch.empty(max(cap, 1) * 24, dtype=torch.uint8, device=dev)
    dense = torch.empty_like(rec)
    cnt = torch.zeros(max(len(n_h), 1), dtype=torch.int32, device=dev)
    cost = torch.empty(max(len(n_h), 1), dtype=torch.float64, device=dev)
    total = torch.zeros(1, dtype=torch.int64, device=dev)
    rod = engine.to_dev(rec_off, dev)
    ms = N.model_struct(model)
    sp = int(torch.cuda.current_stream().cuda_stream)

    def step():
        N.check(lib.bm_mine(C.byref(dc.sent), C.byref(view.docs), n_h.ctypes.data, m_h.ctypes.data,
                            amax.ctypes.data, C.byref(dl.lex), C.byref(ms), 0.5, 0.2,
                            engine._ptr(rod), engine._ptr(rec), engine._ptr(cnt), engine._ptr(cost),
                            sp))
        N.check(lib.bm_compact(engine._ptr(rec), engine._ptr(rod), engine._ptr(cnt), len(n_h),
                               engine._ptr(dense), engine._ptr(total), sp))

    return cuda_ms(step, reps=reps)


def c3(model, n_docs, check_docs):
    g, a, b = synth.c3_shape(n_docs, seed=2026)
    sc = synth.make_corpus(g, a, b, seed=2026)
    c = sc.packed
    plex = sc.world.packed_lexicon()
    dc = engine.DeviceCorpus.upload(c)
    dl = engine.DeviceLexicon.upload(plex)
    view = engine.DocView.of(c)
    cells = int((c.n.astype(np.int64) * c.m).sum())
    res = {}
    ms_host = cuda_ms(lambda: res.__setitem__("r", engine.mine(dc, dl, view, model, 0.5, 0.2)),
                      reps=3)
    recs, cost = res["r"]
    ms = kernel_resident_ms(dc, dl, view, model)
    # parity on a stratified sample: every k-th document, through the oracle
    idx = np.linspace(0, n_docs - 1, min(check_docs, n_docs)).astype(np.int64)
    hb = oracle.HostBatch(c, plex, c.src0[idx], c.n[idx], c.tgt0[idx], c.m[idx])
    want, wcost = oracle.mine(hb, model, 0.5, 0.2, threads=os.cpu_count() or 8)
    sel = np.isin(recs["doc"], idx)
    got = recs[sel].copy()
    got["doc"] = np.searchsorted(idx, got["doc"])
    ok = got.tobytes() == want.tobytes() and np.array_equal(cost[idx].view(np.uint64), wcost.view(np.uint64))
    return {"config": f"C3 skewed corpus, {n_docs} docs", "cells": cells,
            "ms": ms, "doc_pairs_per_s": n_docs / (ms / 1e3), "gcups": cells / (ms / 1e3) / 1e9,
            "timing": "kernel-resident: bm_mine + bm_compact on device buffers (CUDA events)",
            "ms_to_host": ms_host,
            "doc_pairs_per_s_to_host": n_docs / (ms_host / 1e3),
            "records": int(recs.shape[0]),
            "oracle_sample_docs": int(idx.size), "bit_exact_on_sample": bool(ok)}


def c3_full(model, n_docs, chunk, check_per_chunk):
    """C3 at its BASELINE size: n_docs (1M) skewed docs drawn once from
    c3_shape(n_docs, 2026), generated and mined in chunks of `chunk` docs
    (chunk k's text seeded 2026 + k). Per chunk: kernel-resident time
    (bm_mine + bm_compact), time with the records back on the host
    (engine.mine), and an oracle check of a stratified sample."""
    g, a, b = synth.c3_shape(n_docs, seed=2026)
    tot = {"cells": 0, "ms": 0.0, "ms_to_host": 0.0, "records": 0, "checked": 0, "ok": True,
           "gen_s": 0.0, "oracle_s": 0.0}
    for k, lo in enumerate(range(0, n_docs, chunk)):
        hi = min(lo + chunk, n_docs)
        t0 = time.perf_counter()
        sc = synth.make_corpus(g[lo:hi], a[lo:hi], b[lo:hi], seed=2026 + k)
        c = sc.packed
        plex = sc.world.packed_lexicon()
        tot["gen_s"] += time.perf_counter() - t0
        dc = engine.DeviceCorpus.upload(c)
        dl = engine.DeviceLexicon.upload(plex)
        view = engine.DocView.of(c)
        tot["cells"] += int((c.n.astype(np.int64) * c.m).sum())
        res = {}
        tot["ms_to_host"] += cuda_ms(
            lambda: res.__setitem__("r", engine.mine(dc, dl, view, model, 0.5, 0.2)), reps=1)
        recs, cost = res["r"]
        tot["ms"] += kernel_resident_ms(dc, dl, view, model, reps=1)
        tot["records"] += int(recs.shape[0])
        t0 = time.perf_counter()
        # stratified by size: every k-th doc of the size-sorted chunk, plus the largest doc
        order = np.argsort(c.n.astype(np.int64) * c.m, kind="stable")
        idx = np.unique(np.r_[order[np.linspace(0, hi - lo - 1, check_per_chunk).astype(np.int64)]])
        hb = oracle.HostBatch(c, plex, c.src0[idx], c.n[idx], c.tgt0[idx], c.m[idx])
        want, wcost = oracle.mine(hb, model, 0.5, 0.2, threads=os.cpu_count() or 8)
        sel = np.isin(recs["doc"], idx)
        got = recs[sel].copy()
        got["doc"] = np.searchsorted(idx, got["doc"])
        ok = got.tobytes() == want.tobytes() and np.array_equal(cost[idx].view(np.uint64),
                                                                wcost.view(np.uint64))
        tot["oracle_s"] += time.perf_counter() - t0
        tot["ok"] = tot["ok"] and bool(ok)
        tot["checked"] += int(idx.size)
        del dc, dl, view, res, recs, cost, sc, c
        torch.cuda.empty_cache()
        print(json.dumps({"chunk": k, "docs": hi - lo, "ms_so_far": tot["ms"], "ok": tot["ok"]}),
              file=sys.stderr, flush=True)
    ms = tot["ms"]
    return {"config": f"C3 skewed corpus, {n_docs} docs (chunks of {chunk})", "cells": tot["cells"],
            "ms": ms, "doc_pairs_per_s": n_docs / (ms / 1e3), "gcups": tot["cells"] / (ms / 1e3) / 1e9,
            "timing": "kernel-resident: sum over chunks of bm_mine + bm_compact (CUDA events)",
            "ms_to_host": tot["ms_to_host"],
            "doc_pairs_per_s_to_host": n_docs / (tot["ms_to_host"] / 1e3),
            "records": tot["records"], "oracle_sample_docs": tot["checked"],
            "oracle_sample": f"{check_per_chunk} docs per chunk, stratified by n*m incl. the largest",
            "bit_exact_on_sample": tot["ok"], "host_generation_s": tot["gen_s"],
            "oracle_s": tot["oracle_s"]}


def c4(check: bool):
    S = np.random.default_rng(303).random((8192, 8192))
    St, s_off, pitch, n, m = engine.upload_matrices([S])
    res = {}
    ms = cuda_ms(lambda: res.__setitem__("r", engine.nw_paths(St, s_off, pitch, n, m, 0.3)), reps=3)
    cost, paths = res["r"]
    out = {"config": "C4 8192x8192 DP only (random S, seed 303)", "ms_dp_plus_traceback": ms,
           "gcups": 8192 * 8192 / (ms / 1e3) / 1e9}
    if check:
        t0 = time.perf_counter()
        c, ops, _, _ = oracle.nw(S, 0.3)
        out["oracle_s"] = time.perf_counter() - t0
        out["bit_exact"] = bool(c == cost[0] and np.array_equal(ops, paths[0][0]))
    return out


def c5(model, n_docs, check_docs):
    sc = synth.make_corpus(*synth.c2_shape(n_docs), seed=55)
    c = sc.packed
    plex = sc.world.packed_lexicon()
    pens = [0.05, 0.1, 0.2, 0.3, 0.4, 0.6, 0.8, 1.6]
    thrs = [0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9]
    keys = [np.asarray(gd[:, 0] * int(c.m[d]) + gd[:, 1], np.int64) for d, gd in enumerate(sc.gold)]
    dc = engine.DeviceCorpus.upload(c)
    dl = engine.DeviceLexicon.upload(plex)
    view = engine.DocView.of(c)
    res = {}
    ms_call = cuda_ms(lambda: res.__setitem__("r", engine.tune_counts(dc, dl, view, model, pens, thrs, keys)),
                      reps=2)
    p, h = res["r"]
    gold = engine.DeviceGold.of(keys)
    ms = cuda_ms(lambda: engine.tune_counts_device(dc, dl, view, model, pens, thrs, gold), reps=3)
    k = min(check_docs, n_docs)
    hb = oracle.HostBatch(c, plex, c.src0[:k], c.n[:k], c.tgt0[:k], c.m[:k])
    wp, wh = oracle.tune(hb, model, pens, thrs, keys[:k], threads=os.cpu_count() or 8)
    sub = engine.DocView.upload(c.src0[:k], c.n[:k], c.tgt0[:k], c.m[:k])
    sp, sh = engine.tune_counts(dc, dl, sub, model, pens, thrs, keys[:k])
    cells = int((c.n.astype(np.int64) * c.m).sum())
    return {"config": f"C5 tune sweep {n_docs} docs x 64 grid points", "ms": ms,
            "timing": "device-resident: bm_tune with gold keys already on the device (CUDA events)",
            "ms_with_host_gold_packing": ms_call,
            "doc_pairs_per_s": n_docs / (ms / 1e3), "dp_gcups": cells * len(pens) / (ms / 1e3) / 1e9,
            "oracle_sample_docs": k, "counts_identical_on_sample": bool(np.array_equal(sp, wp) and np.array_equal(sh, wh))}


def c5w(model, n_docs):
    """C5 worst case: 64 distinct penalties x 1 threshold."""
    sc = synth.make_corpus(*synth.c2_shape(n_docs), seed=55)
    c = sc.packed
    plex = sc.world.packed_lexicon()
    pens = [0.025 * (k + 1) for k in range(64)]
    keys = [np.asarray(gd[:, 0] * int(c.m[d]) + gd[:, 1], np.int64) for d, gd in enumerate(sc.gold)]
    dc = engine.DeviceCorpus.upload(c)
    dl = engine.DeviceLexicon.upload(plex)
    view = engine.DocView.of(c)
    gold = engine.DeviceGold.of(keys)
    ms = cuda_ms(lambda: engine.tune_counts_device(dc, dl, view, model, pens, [0.5], gold), reps=2)
    cells = int((c.n.astype(np.int64) * c.m).sum())
    return {"config": f"C5 worst case: {n_docs} docs x 64 penalties x 1 threshold", "ms": ms,
            "doc_pairs_per_s": n_docs / (ms / 1e3), "dp_gcups": cells * 64 / (ms / 1e3) / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c3-docs", type=int, default=100000)
    ap.add_argument("--c5-docs", type=int, default=20000)
    ap.add_argument("--check-docs", type=int, default=300)
    ap.add_argument("--c4-check", action="store_true")
    ap.add_argument("--c3-full-docs", type=int, default=1000000)
    ap.add_argument("--c3-chunk", type=int, default=100000)
    ap.add_argument("--check-per-chunk", type=int, default=100)
    ap.add_argument("--only", default="c1,c3,c4,c5")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    model = bm.load_model(MODEL)
    lex = bm.load_lexicon(os.path.join(ROOT, "tests", "golden", "lex5k.tsv"), "xx", "yy")
    todo = args.only.split(",")
    if "c1" in todo:
        print(json.dumps(c1(model, lex)), flush=True)
    if "c3" in todo:
        print(json.dumps(c3(model, args.c3_docs, args.check_docs)), flush=True)
    if "c3full" in todo:
        print(json.dumps(c3_full(model, args.c3_full_docs, args.c3_chunk, args.check_per_chunk)),
              flush=True)
    if "c4" in todo:
        print(json.dumps(c4(args.c4_check)), flush=True)
    if "c5" in todo:
        print(json.dumps(c5(model, args.c5_docs, args.check_docs)), flush=True)
    if "c5w" in todo:
        print(json.dumps(c5w(model, args.c5_docs)), flush=True)


if __name__ == "__main__":
    main()
