"""Reader test corpus (METIS and edge lists): valid files exercising every rule
of H/io.hpp:83-237 and one file per error the reference raises.  Each case is
(name, kind, text bytes, merge_duplicates)."""
import numpy as np


def metis_text(n, rows, weighted, m=None, comments=(), trailing="", eol="\n", final_newline=True):
    """rows[u] = [(v0, w), ...] 0-based; written 1-based like io::write_metis."""
    if m is None:
        und = set()
        for u, r in enumerate(rows):
            for v, _ in r:
                und.add((min(u, v), max(u, v)))
        m = len(und)
    lines = list(comments)
    lines.append(f"{n} {m}" + (" 1" if weighted else ""))
    for r in rows:
        toks = []
        for v, w in r:
            toks.append(str(v + 1))
            if weighted:
                toks.append(w if isinstance(w, str) else repr(float(w)))
        lines.append(" ".join(toks))
    s = eol.join(lines) + (eol if final_newline else "") + trailing
    return s.encode()


def random_graph(rng, n, p, weighted, loops=0.05):
    rows = [[] for _ in range(n)]
    for u in range(n):
        for v in range(u, n):
            if (v == u and rng.random() < loops) or (v != u and rng.random() < p):
                w = float(rng.integers(1, 9)) / 4 if weighted else 1.0
                rows[u].append((v, w))
                if v != u:
                    rows[v].append((u, w))
    for r in rows:
        rng.shuffle(r)  # the reader sorts
    return rows


def cases():
    rng = np.random.default_rng(7)
    out = []
    M = lambda name, text: out.append((name, "metis", text, False))  # noqa: E731
    E = lambda name, text, merge=False: out.append((name, "edges", text, merge))  # noqa: E731
    # ---- valid METIS
    M("tri", b"3 3\n2 3\n1 3\n1 2\n")
    M("tri_weighted", b"3 3 1\n2 1.5 3 2\n1 1.5 3 0.25\n1 2 2 0.25\n")
    M("fmt0", b"3 1 0\n2\n1\n\n")
    M("comments", b"% hello\n%\n3 2\n% inside\n2\n1 3\n2\n")
    M("loop_isolated", b"4 2\n1 2\n1\n\n\n")
    M("no_final_newline", b"2 1\n2\n1")
    M("crlf", b"3 2\r\n2\r\n1 3\r\n2\r\n")
    M("tabs_spaces", b"  3\t 2  \n\t2 \n 1\t3\n2\n")
    M("trailing_blank", b"2 1\n2\n1\n   \nextra junk ignored after the checked line\n")
    M("trailing_comment_then_blank", b"2 1\n2\n1\n% c\n\n")
    M("exp_weights", b"2 1 1\n2 1e-3\n1 0.001\n")
    M("inf_weight", b"2 1 1\n2 inf\n1 INF\n")
    M("zero_nodes", b"0 0\n")
    M("big_ids_order", b"5 4\n5 2\n1\n4\n3 5\n4 1\n")
    for i in range(6):
        n = int(rng.integers(5, 60))
        weighted = bool(i % 2)
        M(f"random{i}", metis_text(n, random_graph(rng, n, 0.15, weighted), weighted))
    # ---- METIS errors (message categories follow H/io.hpp)
    M("err_empty", b"")
    M("err_only_comments", b"% a\n% b\n")
    M("err_header_1tok", b"3\n")
    M("err_header_4tok", b"3 2 1 1\n2\n1 3\n2\n")
    M("err_header_malformed", b"3 x\n2\n1 3\n2\n")
    M("err_fmt_node_weights", b"3 2 10\n2\n1 3\n2\n")
    M("err_missing_lines", b"3 2\n2\n1 3\n")
    M("err_dangling", b"2 1 1\n2\n1 1\n")
    M("err_id_zero", b"2 1\n0\n1\n")
    M("err_id_range", b"2 1\n3\n1\n")
    M("err_id_malformed", b"2 1\n2x\n1\n")
    M("err_id_negative", b"2 1\n-2\n1\n")
    M("err_weight_malformed", b"2 1 1\n2 1.5.2\n1 1\n")
    M("err_weight_zero", b"2 1 1\n2 0\n1 0\n")
    M("err_weight_negative", b"2 1 1\n2 -1\n1 -1\n")
    M("err_weight_nan", b"2 1 1\n2 nan\n1 nan\n")
    M("err_trailing", b"2 1\n2\n1\n3\n")
    M("err_asym_missing", b"3 2\n2 3\n1\n\n")
    M("err_asym_weight", b"2 1 1\n2 1\n1 2\n")
    M("err_duplicate", b"2 1\n2 2\n1 1\n")
    M("err_m_mismatch", b"3 5\n2\n1 3\n2\n")
    M("err_token_before_missing", b"3 2\n9\n")
    # ---- valid edge lists
    E("el_basic", b"0 1\n1 2\n2 0\n")
    E("el_comments", b"# header\n10 20 # tail\n20 30\n\n   # only comment\n30 10\n")
    E("el_weights", b"5 7 0.5\n7 9 2\n9 5 1e1\n")
    E("el_mixed_weights", b"1 2\n2 3 2.5\n")
    E("el_big_ids", b"18446744073709551615 0\n0 9223372036854775808\n")
    E("el_loops", b"4 4\n4 5\n")
    E("el_merge", b"1 2 1\n2 1 2\n1 2 0.5\n", True)
    E("el_merge_unweighted", b"1 2\n2 1\n", True)
    E("el_hash_in_token", b"1 2#x\n2 3\n")
    E("el_empty", b"")
    E("el_no_newline", b"3 4")
    for i in range(4):
        m = int(rng.integers(10, 200))
        ids = rng.integers(0, 1 << 40, size=30)
        lines = []
        seen = set()
        for _ in range(m):
            a, b = int(ids[rng.integers(0, 30)]), int(ids[rng.integers(0, 30)])
            if (min(a, b), max(a, b)) in seen:
                continue
            seen.add((min(a, b), max(a, b)))
            lines.append(f"{a} {b}" + (f" {float(rng.integers(1, 5)) / 2}" if i % 2 else ""))
        E(f"el_random{i}", ("\n".join(lines) + "\n").encode())
    # ---- edge-list errors
    E("el_err_one_token", b"1 2\n3\n")
    E("el_err_four_tokens", b"1 2 3 4\n")
    E("el_err_malformed_u", b"a 2\n")
    E("el_err_malformed_v", b"1 2.0\n")
    E("el_err_weight", b"1 2 x\n")
    E("el_err_weight_zero", b"1 2 0\n")
    E("el_err_duplicate", b"1 2\n2 1\n")
    E("el_err_overflow", b"18446744073709551616 1\n")
    return out


def category(msg: str) -> str:
    """Coarse class of a reader error message (device and reference word some differently)."""
    keys = ["unexpected end of file", "malformed header", "unsupported fmt", "adjacency lines, got",
            "dangling weight", "out of range", "malformed integer", "malformed weight", "nonpositive",
            "trailing content", "asymmetric", "duplicate", "header promises", "expected 'u v [w]'"]
    for k in keys:
        if k in msg:
            return k
    return "other:" + msg
