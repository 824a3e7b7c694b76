"""Generates tests/golden/* from the UNMODIFIED reference.

Run in the build container (needs /root/reference to build oracle/_ref):
    make -C oracle && python tests/golden/make_golden.py

Every vector is produced by the reference's own public API through
oracle/_ref/libcommdet_ref.so (oracle/ref_capi.cpp):
  Graph::from_edges, generate_planted, modularity, coverage, dominant_label,
  coarsen, Partition::compacted, combine_hashed, djb2, delta_mod,
  run_plp / run_plm / run_plmr / run_epp (workers = 1, deterministic).
Random instances come from numpy's seeded PCG64 (weights are integers 1..5 or
dyadic fp32 values so fp32 device storage is exact).  The fixtures let the
CPU suite pin the C oracle without the reference and travel to the GPU box.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle import oracle as O  # noqa: E402


def rand_edges(rng, n, p, weights="int", loop_p=0.0):
    eu, ev, ew = [], [], []
    for u in range(n):
        for v in range(u + 1, n):
            if rng.random() < p:
                eu.append(u)
                ev.append(v)
                ew.append(_w(rng, weights))
        if loop_p > 0 and rng.random() < loop_p:
            eu.append(u)
            ev.append(u)
            ew.append(_w(rng, weights))
    if not eu:
        eu, ev, ew = [0], [min(1, n - 1)], [1.0]
    return np.array(eu, np.int32), np.array(ev, np.int32), np.array(ew, np.float64)


def _w(rng, kind):
    if kind == "unit":
        return 1.0
    if kind == "int":
        return float(rng.integers(1, 6))
    return float((int(rng.integers(0, 1 << 24)) + 1) * 2.0 ** -24)  # dyadic, exact in fp32


def main():
    rng = np.random.default_rng(20261019)
    arrays = {}
    cases = []
    # ---- random instances ----------------------------------------------------
    for i in range(40):
        n = int(rng.integers(4, 61))
        kind = ["unit", "int", "dyadic"][i % 3]
        eu, ev, ew = rand_edges(rng, n, float(rng.uniform(0.08, 0.4)), kind, loop_p=0.15 if i % 2 else 0.0)
        edges = list(zip(eu.tolist(), ev.tolist(), ew.tolist()))
        rg = O.RefGraph.from_edges(n, edges)
        csr = rg.csr()
        k = int(rng.integers(1, 7))
        z = rng.integers(0, k, size=n).astype(np.int32)
        zc, _ = O.ref_compacted(z)
        key = f"r{i}"
        arrays[f"{key}_eu"], arrays[f"{key}_ev"], arrays[f"{key}_ew"] = eu, ev, ew
        arrays[f"{key}_off"], arrays[f"{key}_col"], arrays[f"{key}_w"] = csr.off, csr.col, csr.w
        arrays[f"{key}_vol"], arrays[f"{key}_loop"] = csr.vol, csr.loop
        arrays[f"{key}_z"], arrays[f"{key}_zc"] = z, zc
        mods = {}
        for gamma in (0.0, 0.5, 1.0, 2.0):
            q, cov = rg.modularity(z, gamma, ub=k)
            mods[str(gamma)] = q
        # one synchronous sweep from singletons and from z
        for tag, lab in (("s", np.arange(n, dtype=np.int32)), ("z", z)):
            out = np.array([rg.dominant_label(lab, u) if csr.off[u + 1] > csr.off[u] else lab[u]
                            for u in range(n)], np.int32)
            arrays[f"{key}_sweep_{tag}"] = out
        cg, pi = rg.coarsen(zc)
        cc = cg.csr()
        arrays[f"{key}_coff"], arrays[f"{key}_ccol"], arrays[f"{key}_cw"] = cc.off, cc.col, cc.w
        arrays[f"{key}_cvol"], arrays[f"{key}_cloop"] = cc.vol, cc.loop
        u = int(rng.integers(0, n))
        t = int(z[int(rng.integers(0, n))])
        delta = {str(g): rg.delta_mod(z, u, t, g, ub=k) for g in (0.0, 0.5, 1.0, 2.0 * csr.total)}
        plp, plp_rep, plp_trace = rg.run_plp(theta=0, workers=1)
        plm, plm_rep = rg.run_louvain(refine=False, workers=1)
        plmr, plmr_rep = rg.run_louvain(refine=True, workers=1)
        arrays[f"{key}_plp"], arrays[f"{key}_plm"], arrays[f"{key}_plmr"] = plp, plm, plmr
        cases.append(dict(key=key, n=n, k=k, m=csr.m, total=csr.total, modularity=mods,
                          coverage=rg.modularity(z, 1.0, ub=k)[1], cm=cg.info()[2], ctotal=cg.info()[3],
                          delta_u=u, delta_t=t, delta=delta, plp_q=plp_rep["modularity"],
                          plp_iters=plp_rep["iterations"], plm_q=plm_rep["modularity"],
                          plmr_q=plmr_rep["modularity"], stable=rg.is_stable(plp)))
    # ---- planted generator ----------------------------------------------------
    planted = []
    for spec in [(6, 2, 1.0, 0.0, 1), (300, 5, 0.2, 0.01, 7), (2000, 8, 0.05, 0.002, 3), (103, 10, 0.0, 0.0, 1),
                 (1000, 10, 0.1, 0.002, 1)]:
        rg, truth = O.RefGraph.planted(*spec, workers=1)
        c = rg.csr()
        key = "p_" + "_".join(str(x) for x in spec)
        arrays[f"{key}_off"], arrays[f"{key}_col"], arrays[f"{key}_truth"] = c.off, c.col, truth
        planted.append(dict(key=key, spec=list(spec), m=c.m))
    # ---- ensemble --------------------------------------------------------------
    sols = [rng.integers(0, 3, size=37).astype(np.int32) for _ in range(4)]
    for j, s in enumerate(sols):
        arrays[f"ens_sol{j}"] = s
    arrays["ens_hashed"] = O.ref_combine_hashed(sols)
    arrays["ens_exact"] = O.ref_combine_exact(sols)
    djb = {"": O.ref_djb2(b""), "01": O.ref_djb2(bytes([1])), "0102ff": O.ref_djb2(bytes([1, 2, 255]))}
    manifest = dict(cases=cases, planted=planted, djb2=djb,
                    generator="tests/golden/make_golden.py via oracle/_ref (reference headers, unmodified)")
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays,", len(cases), "random cases")


if __name__ == "__main__":
    main()
