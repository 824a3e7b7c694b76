"""The CLI drop-in (tools/commdet_gpu.cpp) against
the reference library (oracle/_ref): `generate` writes the same METIS bytes as
io::write_metis of generate_planted; `detect --community-graph` writes the
same bytes as io::write_community_graph of the best partition; `score` prints
the reference's graph_rand_index; `detect --report` carries
RunReport::to_json's fields (H/report.hpp:42-70); exit codes follow
P/tools/commdet.cpp:24-25."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cli(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("cli") / "commdet_gpu")
    lib_dir = os.path.join(ROOT, "paper_1304_4453_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tools", "commdet_gpu.cpp"), "-o", exe, "-L" + lib_dir, "-lcommdet_cuda",
                    "-Wl,-rpath," + lib_dir], check=True)
    return exe


def run(cli, *args, ok=True):
    r = subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=300)
    if ok:
        assert r.returncode == 0, r.stdout + r.stderr
    return r


def kv(text):
    out = {}
    for line in text.splitlines():
        parts = line.split()
        if len(parts) == 2:
            out[parts[0]] = parts[1]
    return out


def test_generate_matches_reference_writer(cli, ref, tmp_path):
    g_path, t_path = tmp_path / "g.metis", tmp_path / "truth.txt"
    out = kv(run(cli, "generate", "--n", 3000, "--k", 30, "--pin", 0.1, "--pout", 0.002, "--seed", 7,
                 "--output", g_path, "--ground-truth", t_path).stdout)
    rg, truth = ref.RefGraph.planted(3000, 30, 0.1, 0.002, 7)
    r_path = tmp_path / "r.metis"
    rg.write_metis(r_path)
    assert g_path.read_bytes() == r_path.read_bytes()
    assert int(out["nodes"]) == 3000 and int(out["edges"]) == rg.info()[2] and int(out["blocks"]) == 30
    z = np.loadtxt(t_path, dtype=np.int64)
    assert len(z) == 3000 and z.min() == 0


def test_detect_report_and_outputs(cli, ref, tmp_path):
    g_path = tmp_path / "g.metis"
    run(cli, "generate", "--n", 2000, "--k", 20, "--pin", 0.2, "--pout", 0.003, "--output", g_path)
    rep, part, cg = tmp_path / "rep.json", tmp_path / "z.txt", tmp_path / "cg.metis"
    out = kv(run(cli, "detect", "--algo", "plmr", "--input", g_path, "--runs", 2, "--report", rep, "--output", part,
                 "--community-graph", cg).stdout)
    assert out["algorithm"] == "plmr" and out["runs"] == "2"
    j = json.loads(rep.read_text())
    assert set(j) == {"average", "best_modularity", "runs"}
    assert set(j["average"]) == {"time_ms", "modularity", "coverage"}
    r0 = j["runs"][0]
    for k in ("algorithm", "input", "workers", "seed", "total_ms", "modularity", "coverage", "communities", "levels"):
        assert k in r0
    assert set(r0["levels"][0]) == {"move_ms", "coarsen_ms", "refine_ms"}
    assert [r["seed"] for r in j["runs"]] == [1, 2]
    assert float(out["best_modularity"]) == pytest.approx(max(r["modularity"] for r in j["runs"]), rel=1e-12)
    z = np.loadtxt(part, dtype=np.int32)
    assert int(out["communities"]) == z.max() + 1
    # community graph: byte-identical to the reference's writer on the same partition
    rg = ref.RefGraph.read_metis(str(g_path))
    r_cg = tmp_path / "rcg.metis"
    rg.write_community_graph(z, r_cg)
    assert cg.read_bytes() == r_cg.read_bytes()
    assert (tmp_path / "cg.metis.sizes").read_bytes() == (tmp_path / "rcg.metis.sizes").read_bytes()
    # PLP and EPP reports carry iterations / phases
    run(cli, "detect", "--algo", "plp", "--shuffle", "--input", g_path, "--report", rep)
    assert "iterations" in json.loads(rep.read_text())["runs"][0]
    run(cli, "detect", "--algo", "epp", "--input", g_path, "--report", rep)
    assert set(json.loads(rep.read_text())["runs"][0]["phases"]) == {"base_ms", "combine_ms", "coarsen_ms",
                                                                       "final_ms"}


def test_score_rand_index(cli, ref, tmp_path):
    g_path, t_path, z_path = tmp_path / "g.metis", tmp_path / "t.txt", tmp_path / "z.txt"
    run(cli, "generate", "--n", 2500, "--k", 25, "--pin", 0.15, "--pout", 0.004, "--output", g_path,
        "--ground-truth", t_path)
    run(cli, "detect", "--algo", "plm", "--input", g_path, "--output", z_path)
    out = kv(run(cli, "score", "--input", g_path, "--partition", z_path, "--reference", t_path).stdout)
    rg = ref.RefGraph.read_metis(str(g_path))
    z = np.loadtxt(z_path, dtype=np.int32)
    t = np.loadtxt(t_path, dtype=np.int32)
    assert float(out["rand_index"]) == pytest.approx(rg.rand_index(z, t), rel=1e-15)
    q, cov = rg.modularity(z)
    assert float(out["modularity"]) == pytest.approx(q, rel=1e-12)
    assert float(out["coverage"]) == pytest.approx(cov, rel=1e-12)


def test_bench_and_errors(cli, tmp_path):
    data = tmp_path / "b.tsv"
    r = run(cli, "bench", "--mode", "weak", "--algo", "plm", "--gen-n", 2000, "--gen-k", 20, "--gen-pin", 0.1,
            "--gen-pout", 0.002, "--threads-list", "1,2", "--data", data)
    lines = r.stdout.strip().splitlines()
    assert lines[0].split() == ["threads", "time_ms", "speedup", "modularity", "edges"]
    assert len(lines) == 3 and data.read_text().startswith("threads\ttime_ms")
    e = run(cli, "detect", "--input", tmp_path / "missing.metis", ok=False)
    assert e.returncode == 2 and "error: cannot open" in e.stderr
    e = run(cli, "detect", "--algo", "xyz", "--input", tmp_path / "b.tsv", ok=False)
    assert e.returncode == 2
    e = run(cli, "bench", "--mode", "weak", ok=False)
    assert e.returncode == 2 and "weak scaling requires" in e.stderr
    e = run(cli, "frobnicate", ok=False)
    assert e.returncode == 2
