"""The C-ABI library loads and exports every symbol include/commdet_cuda.h
declares (CPU only: no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def header_symbols():
    with open(os.path.join(ROOT, "include", "commdet_cuda.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"CD_API\s+[\w\s\*]+?\b(cd_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = header_symbols()
    for s in ["cd_plp_run", "cd_louvain_run", "cd_epp_run", "cd_modularity", "cd_coarsen", "cd_prolong",
              "cd_plp_sweep_sync", "cd_move_eval", "cd_combine_hashed", "cd_graph_from_edges"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    import paper_1304_4453_b200 as P
    lib = P.load_library()
    for s in header_symbols():
        assert hasattr(lib, s), s
    assert sorted(P.EXPORTS) == header_symbols()
    out = subprocess.run(["nm", "-D", "--defined-only", P.library_path()], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert set(header_symbols()) <= exported
    # nothing but the C ABI leaks out of the library
    assert all(s.startswith("cd_") for s in exported), sorted(s for s in exported if not s.startswith("cd_"))[:5]


def test_version_and_config_defaults():
    import paper_1304_4453_b200 as P
    lib = P.load_library()
    assert b"sm_100a" in lib.cd_version()
    c = P._LouvainConfig()
    lib.cd_louvain_config_default(ctypes.byref(c))
    assert c.gamma == 1.0 and c.max_move_iterations == 32 and c.max_levels == 64  # H/louvain.hpp:15-22
    p = P._PlpConfig()
    lib.cd_plp_config_default(ctypes.byref(p))
    assert p.theta == -1 and p.max_iterations == 100  # H/plp.hpp:16-22
    e = P._EnsembleConfig()
    lib.cd_ensemble_config_default(ctypes.byref(e))
    assert e.ensemble_size == 4 and e.base == P.ALGO_PLP and e.final_algo == P.ALGO_PLMR  # H/ensemble.hpp:19-31
    assert e.base_plp.randomize_order == 1


def test_python_struct_layout_matches_header():
    """ctypes mirrors must match the C layout (compiled probe)."""
    import paper_1304_4453_b200 as P
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "commdet_cuda.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(cd_plp_config), sizeof(cd_louvain_config),
         sizeof(cd_ensemble_config), sizeof(cd_report), sizeof(cd_graph_info), sizeof(cd_lfr_spec),
         sizeof(cd_kernel_stat));
  return 0;
}
'''
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "probe.c")
        with open(c, "w") as f:
            f.write(src)
        exe = os.path.join(d, "probe")
        subprocess.run(["gcc", "-I" + os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        sizes = [int(x) for x in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    mine = [ctypes.sizeof(t) for t in (P._PlpConfig, P._LouvainConfig, P._EnsembleConfig, P._Report, P._GraphInfo,
                                       P._LfrSpec, P._KStat)]
    assert mine == sizes


def test_no_gpu_fails_loudly():
    """Without a device the product raises; there is no CPU fallback."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1304_4453_b200 as P
    with pytest.raises(P.CudaError):
        P.Context(0)
