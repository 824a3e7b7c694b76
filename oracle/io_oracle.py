"""CPU restatement of the reference's text readers (TEST INFRASTRUCTURE ONLY).

    read_metis      H/io.hpp:83-165
    read_edge_list  H/io.hpp:190-237

Pure Python (small inputs): the checker for the device readers
(cd_graph_read_metis / cd_graph_read_edge_list).  It is itself pinned against
the unmodified reference (oracle/_ref ref_read_metis / ref_read_edge_list) by
tests/test_io_oracle.py.  Errors raise InputError with the reference's message.
"""
import re

import numpy as np

from . import oracle as O


class InputError(ValueError):
    pass


_WS = " \t\n\v\f\r"
_FLOAT = re.compile(r"-?(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?")
_SPECIAL = re.compile(r"-?(?:inf|infinity|nan(?:\([A-Za-z0-9_]*\))?)", re.IGNORECASE)


def split_ws(line: str):
    """detail::split_ws (H/io.hpp:39-52)."""
    out, i = [], 0
    while i < len(line):
        while i < len(line) and line[i] in _WS:
            i += 1
        j = i
        while j < len(line) and line[j] not in _WS:
            j += 1
        if j > i:
            out.append(line[i:j])
        i = j
    return out


def parse_uint(tok: str, ctx: str) -> int:
    """detail::parse_uint (H/io.hpp:54-60): std::from_chars(uint64)."""
    if not tok or any(c not in "0123456789" for c in tok) or int(tok) >= 1 << 64:
        raise InputError(f"malformed integer '{tok}' in {ctx}")
    return int(tok)


def parse_weight(tok: str, ctx: str) -> float:
    """detail::parse_weight (H/io.hpp:62-68): std::from_chars(double), general format."""
    if _FLOAT.fullmatch(tok):
        return float(tok)
    if _SPECIAL.fullmatch(tok):
        t = tok.lower().lstrip("-")
        v = float("nan") if t.startswith("nan") else float("inf")
        return -v if tok.startswith("-") else v
    raise InputError(f"malformed weight '{tok}' in {ctx}")


def _lines(data: bytes):
    """std::getline over the whole text: '\\n'-separated, no empty line after a final '\\n'."""
    text = data.decode("latin-1")
    parts = text.split("\n")
    if parts and parts[-1] == "" and text.endswith("\n"):
        parts.pop()
    if text == "":
        parts = []
    return parts


def read_metis(data: bytes, path: str = "<metis>"):
    """Returns (n, edges [(u, v, w)] with v >= u, m) -> built by from_edges; raises InputError."""
    lines = _lines(data)
    pos = 0
    lineno = 0

    def next_line(required):
        nonlocal pos, lineno
        while pos < len(lines):
            line = lines[pos]
            pos += 1
            lineno += 1
            if line and line[0] == "%":
                continue
            return line
        if required:
            raise InputError(f"{path}: unexpected end of file")
        return None

    header = split_ws(next_line(True))
    if len(header) < 2 or len(header) > 3:
        raise InputError(f"{path}: malformed header")
    n = parse_uint(header[0], path + " header")
    m = parse_uint(header[1], path + " header")
    weighted = False
    if len(header) == 3:
        fmt = parse_uint(header[2], path + " header")
        if fmt == 1:
            weighted = True
        elif fmt != 0:
            raise InputError(f"{path}: unsupported fmt code {fmt} (node weights are not supported)")
    adj = [[] for _ in range(n)]
    for u in range(n):
        line = next_line(False)
        if line is None:
            raise InputError(f"{path}: expected {n} adjacency lines, got {u}")
        toks = split_ws(line)
        stride = 2 if weighted else 1
        if len(toks) % stride:
            raise InputError(f"{path}:{lineno}: dangling weight token")
        for i in range(0, len(toks), stride):
            v1 = parse_uint(toks[i], f"{path}:{lineno}")
            if v1 < 1 or v1 > n:
                raise InputError(f"{path}:{lineno}: neighbor id {v1} out of range")
            w = parse_weight(toks[i + 1], f"{path}:{lineno}") if weighted else 1.0
            if not w > 0.0:
                raise InputError(f"{path}:{lineno}: nonpositive edge weight")
            adj[u].append((v1 - 1, w))
    line = next_line(False)
    if line is not None and split_ws(line):
        raise InputError(f"{path}: trailing content after {n} adjacency lines")
    for u in range(n):
        adj[u].sort()
    edges = []
    for u in range(n):
        for v, w in adj[u]:
            if v < u:
                continue
            edges.append((u, v, w))
            if v != u:
                rev = [x for x in adj[v] if x[0] == u]
                if not rev or rev[0][1] != w:  # lower_bound(u, 0.0): v's smallest weight towards u
                    raise InputError(f"{path}: asymmetric adjacency between nodes {u + 1} and {v + 1}")
    g = build(n, edges, False)
    if g.m != m:
        raise InputError(f"{path}: header promises {m} edges, file contains {g.m}")
    return g, weighted


def read_edge_list(data: bytes, merge_duplicates=False, path: str = "<edge list>"):
    """Returns (CSR, original ids); raises InputError."""
    raw = []
    any_w = False
    for lineno, line in enumerate(_lines(data), start=1):
        h = line.find("#")
        toks = split_ws(line if h < 0 else line[:h])
        if not toks:
            continue
        if len(toks) not in (2, 3):
            raise InputError(f"{path}:{lineno}: expected 'u v [w]'")
        ctx = f"{path}:{lineno}"
        u = parse_uint(toks[0], ctx)
        v = parse_uint(toks[1], ctx)
        w = parse_weight(toks[2], ctx) if len(toks) == 3 else 1.0
        any_w |= len(toks) == 3
        if not w > 0.0:
            raise InputError(f"{ctx}: nonpositive edge weight")
        raw.append((u, v, w))
    original = sorted({x for e in raw for x in e[:2]})
    remap = {x: i for i, x in enumerate(original)}
    edges = [(remap[u], remap[v], w) for u, v, w in raw]
    return build(len(original), edges, merge_duplicates), np.array(original, np.uint64), any_w


def build(n, edges, merge):
    """Graph::from_edges through the C oracle (H/graph.hpp:48-81); the duplicate
    check restates sort_and_merge's message (H/graph.hpp:169-181)."""
    if not merge:
        rows = [[] for _ in range(n)]
        for u, v, _ in edges:
            rows[u].append(v)
            if v != u:
                rows[v].append(u)
        for u in range(n):
            r = sorted(rows[u])
            for i in range(len(r) - 1):
                if r[i] == r[i + 1]:
                    raise InputError(f"duplicate edge {u},{r[i]}")
    if not edges:
        return O.from_arrays(n, np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0), merge)
    eu = np.array([e[0] for e in edges], np.int64)
    ev = np.array([e[1] for e in edges], np.int64)
    ew = np.array([e[2] for e in edges], np.float64)
    try:
        return O.from_arrays(n, eu, ev, ew, merge)
    except O.OracleError as exc:  # duplicates etc. are input errors of the reader
        raise InputError(str(exc)) from exc
