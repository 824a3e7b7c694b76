"""Caches the UNMODIFIED reference's end-to-end results on the headline graphs.

    make -C oracle && python tests/golden/make_ref_quality.py [--only KEY ...] [--runs R]

The reference's run_plp / run_plm / run_plmr / run_epp (oracle/_ref, built
from /root/reference by oracle/Makefile) run on the IDENTICAL bytes the
device builds: the graph comes from the C port of the seeded generators
(oracle/commdet_oracle.c), which tests/test_gpu_parity.py and bench.py check
byte-for-byte against the device generator.  The reference takes minutes per
run at C3 (PLM 624 s on 8 threads), far too long for the GPU
test suite, so its modularity / community count are cached here once
 and the -m gpu tests compare the device run against them
(tests/test_gpu_headline.py).

Settings (SURVEY.md 8(c) "End-to-end oracle"):
  PLP   randomize_order=true, seed=1, workers=1 (the named parity setting;
        deterministic) -- plus the default order with all host threads.
  PLM / PLMR / EPP  workers = all host threads; R runs, median Q recorded
        (multi-thread output varies run to run, R/SPEC.md:243, :349).

Output: tests/golden/ref_quality.json, keyed "<workload>/<setting>" with the
graph's n, m, D and a checksum of its columns, so a test can verify it is
comparing against the same bytes.  Written after every run (partial progress
survives an interrupt).
"""
import argparse
import hashlib
import json
import os
import platform
import statistics
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

OUT = os.path.join(HERE, "ref_quality.json")

GRAPHS = {
    "c1": dict(gen="planted"),
    "c2": dict(gen="lfr"),
    "c3": dict(gen="rmat", scale=24, weighted=False),
    "c4": dict(gen="rmat", scale=22, weighted=True),
}

# key -> (graph, algo, setting)
JOBS = {
    "c1_planted_plp/parity": ("c1", "plp", "parity"),
    "c1_planted_plm/threads": ("c1", "plm", "threads"),
    "c2_lfr_plm/threads": ("c2", "plm", "threads"),
    "c3_rmat24_plp/parity": ("c3", "plp", "parity"),
    "c3_rmat24_plp/threads": ("c3", "plp", "threads"),
    "c4_rmat22w_plmr/threads": ("c4", "plmr", "threads"),
    "c4_rmat22w_epp/threads": ("c4", "epp", "threads"),
    "c3_rmat24_plm/threads": ("c3", "plm", "threads"),
}


def graph_digest(g):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(g.off, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(g.col, dtype=np.int32).tobytes())
    return h.hexdigest()[:16]


def make_graph(key):
    spec = GRAPHS[key]
    if spec["gen"] == "planted":
        return O.generate_planted(100000, 1000, 0.1, 2 / 99900, 1)[0]
    if spec["gen"] == "lfr":
        return O.generate_lfr(seed=1)[0]
    return O.generate_rmat(spec["scale"], 16, 0.57, 0.19, 0.19, weighted=spec["weighted"], seed=1)


def run_once(rg, algo, setting, threads):
    if algo == "plp":
        if setting == "parity":
            z, rep, _ = rg.run_plp(randomize=True, seed=1, workers=1)
        else:
            z, rep, _ = rg.run_plp(workers=threads)
    elif algo in ("plm", "plmr"):
        z, rep = rg.run_louvain(refine=algo == "plmr", workers=threads)
    else:
        z, rep = rg.run_epp(workers=threads)
    return rep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--runs", type=int, default=3)
    args = ap.parse_args()
    assert O.ref_available(), "build oracle/_ref first (make -C oracle)"
    res = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            res = json.load(f)
    threads = len(os.sched_getaffinity(0))
    graphs = {}
    for key, (gk, algo, setting) in JOBS.items():
        if args.only and key not in args.only:
            continue
        if gk not in graphs:
            t0 = time.time()
            g = make_graph(gk)
            graphs.clear()  # one graph resident at a time (C3 reference CSR ~ 8 GB)
            graphs[gk] = (g, O.RefGraph.from_csr(g), graph_digest(g), time.time() - t0)
        g, rg, dig, gen_s = graphs[gk]
        runs = 1 if (algo == "plp" and setting == "parity") else args.runs
        reps = []
        for _ in range(runs):
            reps.append(run_once(rg, algo, setting, threads))
            print(key, reps[-1]["modularity"], reps[-1]["community_count"], reps[-1]["total_ms"], flush=True)
        qs = [r["modularity"] for r in reps]
        med = sorted(range(len(reps)), key=lambda i: qs[i])[len(reps) // 2]
        res[key] = {
            "graph": {"n": g.n, "m": g.m, "D": g.D, "digest": dig},
            "algo": algo, "setting": setting,
            "workers": 1 if setting == "parity" else threads,
            "randomize_order": setting == "parity",
            "runs": len(reps), "modularity": qs[med], "modularity_all": qs,
            "communities": reps[med]["community_count"],
            "total_ms": statistics.median(r["total_ms"] for r in reps),
            "host": f"{platform.node()} nproc={threads}",
            "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
        }
        with open(OUT, "w") as f:
            json.dump(res, f, indent=1, sort_keys=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
