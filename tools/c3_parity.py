"""C3 at full size against the CPU oracle.

  records   the 1,000,000-document C3 corpus of bench.py (synth.c3_shape(1M,
            seed 2026), native per-document generator) mined on the GPU
            (engine.mine: bm_mine + bm_compact, forward model): sha256 of the
            whole record stream and of the path costs, against oracle.mine over
            every document (16 host threads).
  stream    the same corpus written as JSONL text and mined end to end by
            mine_corpus_file (streamed chunks, both models, device merge, native
            TSV emission), per-phase timings; the oracle-based emission of the
            same file -- native ingest, oracle.mine in both orientations, the
            host C++ bidirectional_merge + TSV writer (bm_ingest_emit) -- must
            give the same bytes.

Writes one JSON object (profiles/r02_c3_1m_parity.json when run as in
DESIGN.md). Usage: python tools/c3_parity.py [--docs N] [--parts records,stream]
"""

from __future__ import annotations

import argparse
import hashlib
import io
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import numpy as np  # noqa: E402

import oracle  # noqa: E402  (checker only)
import paper_1509_08639_b200 as bm  # noqa: E402
from paper_1509_08639_b200 import engine, synth  # noqa: E402

MODEL_F = os.path.join(ROOT, "tests", "golden", "model5k_fwd.json")
MODEL_B = os.path.join(ROOT, "tests", "golden", "model5k_bwd.json")
SEED = 2026


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()


def part_records(n_docs: int, threads: int) -> dict:
    model = bm.load_model(MODEL_F)
    g, a, b = synth.c3_shape(n_docs, seed=SEED)
    t0 = time.perf_counter()
    sc = synth.make_corpus_native(g, a, b, seed=SEED)
    c = sc.packed
    plex = sc.world.packed_lexicon()
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    recs, cost = engine.mine(engine.DeviceCorpus.upload(c), engine.DeviceLexicon.upload(plex),
                             engine.DocView.of(c), model, 0.5, 0.2)
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    want, wcost = oracle.mine(oracle.HostBatch(c, plex), model, 0.5, 0.2, threads=threads)
    t_cpu = time.perf_counter() - t0
    out = {"docs": int(c.n_docs), "cells": int((c.n.astype(np.int64) * c.m).sum()),
           "records": int(recs.shape[0]),
           "gpu_records_sha256": sha(recs), "oracle_records_sha256": sha(want),
           "gpu_cost_sha256": sha(cost), "oracle_cost_sha256": sha(wcost),
           "generate_s": t_gen, "gpu_mine_to_host_s": t_gpu, "oracle_s": t_cpu,
           "oracle_threads": threads}
    out["identical"] = (out["gpu_records_sha256"] == out["oracle_records_sha256"]
                        and out["gpu_cost_sha256"] == out["oracle_cost_sha256"])
    return out


def part_stream(n_docs: int, threads: int, path: str) -> dict:
    from paper_1509_08639_b200 import ingest
    from paper_1509_08639_b200.ingest import NativeCorpus

    fwd, bwd = bm.load_model(MODEL_F), bm.load_model(MODEL_B)
    lex = synth.SynthWorld(5000).lexicon()
    g, a, b = synth.c3_shape(n_docs, seed=SEED)
    t0 = time.perf_counter()
    synth.write_jsonl_native(path, g, a, b, seed=SEED)
    t_write = time.perf_counter() - t0
    cfg = bm.MinerConfig(bm.MiningParams(0.5, 0.2))

    class Sha:
        def __init__(self):
            self.h = hashlib.sha256()
            self.n = 0
            self.lines = 0

        def write(self, s: str):
            data = s.encode("utf-8")
            self.h.update(data)
            self.n += len(data)
            self.lines += s.count("\n")

    sink = Sha()
    t0 = time.perf_counter()
    rep = bm.mine_corpus_file(path, fwd, bwd, lex, cfg, sink)
    wall = time.perf_counter() - t0
    phases = dict(ingest.LAST_TIMINGS)
    # oracle-based emission of the same file
    t0 = time.perf_counter()
    nc = NativeCorpus.load(path)
    c = nc.packed
    plex = nc.lexicon(lex)
    want_f, _ = oracle.mine(oracle.HostBatch(c, plex), fwd, 0.5, 0.2, threads=threads)
    pb = plex.swapped()
    hb = oracle.HostBatch(c, pb, c.tgt0, c.m, c.src0, c.n)
    want_b, _ = oracle.mine(hb, bwd, 0.5, 0.2, threads=threads)
    k = c.n_docs
    data, orep = nc.emit(want_f, want_b, np.zeros(k, np.uint8), np.ones(k, np.uint8),
                         np.zeros(k, np.uint8))
    t_oracle = time.perf_counter() - t0
    want_sha = hashlib.sha256(data).hexdigest()
    return {"docs": n_docs, "jsonl_bytes": os.path.getsize(path), "write_jsonl_s": t_write,
            "mine_corpus_file_s": wall, "docs_per_s": n_docs / wall, "phases_s": phases,
            "tsv_bytes": sink.n, "tsv_lines": sink.lines, "pairs_emitted": rep.pairs_emitted,
            "tsv_sha256": sink.h.hexdigest(), "oracle_tsv_sha256": want_sha,
            "oracle_pairs": int(orep[0]), "oracle_emission_s": t_oracle,
            "identical": sink.h.hexdigest() == want_sha and sink.n == len(data)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--docs", type=int, default=1_000_000)
    ap.add_argument("--parts", default="records,stream")
    ap.add_argument("--threads", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--jsonl", default="/tmp/c3_1m.jsonl")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    torch.cuda.set_device(0)
    res = {"config": f"C3 {args.docs} docs, seed {SEED}, threshold 0.5, penalty 0.2",
           "host_threads": args.threads}
    parts = args.parts.split(",")
    if "records" in parts:
        res["records"] = part_records(args.docs, args.threads)
        print(json.dumps(res["records"]), file=sys.stderr, flush=True)
    if "stream" in parts:
        res["stream"] = part_stream(args.docs, args.threads, args.jsonl)
        print(json.dumps(res["stream"]), file=sys.stderr, flush=True)
    line = json.dumps(res, indent=1)
    print(line)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(line + "\n")


if __name__ == "__main__":
    main()
