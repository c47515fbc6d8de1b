"""Graph file ingestion (graph.hpp:57-147): whitespace edge lists
("src dst [weight]", '#' comments, node count = max index + 1) and
MatrixMarket coordinate files; edges deduplicated keeping the last weight and
returned in canonical (src, dst) order.  Host-side I/O, not on the device path.
"""
from __future__ import annotations

import numpy as np


def _dedup(src, dst, w):
    # stable sort by (src, dst), keep the last occurrence (graph.hpp:42-55)
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    w = np.asarray(w, np.float64)
    if src.size == 0:
        return src.astype(np.int32), dst.astype(np.int32), w
    order = np.lexsort((np.arange(src.size), dst, src))
    s, d, ww = src[order], dst[order], w[order]
    last = np.ones(s.size, bool)
    last[:-1] = (s[1:] != s[:-1]) | (d[1:] != d[:-1])
    return s[last].astype(np.int32), d[last].astype(np.int32), ww[last]


def load_edge_list(path):
    src, dst, w = [], [], []
    max_idx = -1
    try:
        fh = open(path)
    except OSError:
        raise RuntimeError(f"cannot open {path}") from None
    with fh:
        for line_no, line in enumerate(fh, 1):
            line = line.split("#", 1)[0]
            tok = line.split()
            if not tok:
                continue
            if len(tok) < 2:
                raise RuntimeError(f"{path}:{line_no}: expected 'src dst [weight]'")
            if len(tok) > 3:
                raise RuntimeError(f"{path}:{line_no}: trailing tokens")
            s, d = int(tok[0]), int(tok[1])
            if s < 0 or d < 0:
                raise RuntimeError(f"{path}:{line_no}: negative node index")
            src.append(s)
            dst.append(d)
            w.append(float(tok[2]) if len(tok) == 3 else 1.0)
            max_idx = max(max_idx, s, d)
    s, d, ww = _dedup(src, dst, w)
    return {"n": max_idx + 1, "src": s, "dst": d, "weight": ww}


def load_matrix_market(path):
    try:
        fh = open(path)
    except OSError:
        raise RuntimeError(f"cannot open {path}") from None
    with fh:
        lines = fh.read().splitlines()
    if not lines:
        raise RuntimeError(f"{path}: empty file")
    head = lines[0].split()
    if len(head) < 4 or head[0] != "%%MatrixMarket" or head[1] != "matrix" or \
            head[2] != "coordinate":
        raise RuntimeError(f"{path}:1: expected a MatrixMarket coordinate header")
    field = head[3]
    symmetry = head[4] if len(head) > 4 else "general"
    pattern = field == "pattern"
    symmetric = symmetry in ("symmetric", "skew-symmetric")
    if field not in ("real", "integer") and not pattern:
        raise RuntimeError(f"{path}:1: unsupported field type '{field}'")
    i = 1
    while i < len(lines) and (not lines[i] or lines[i][0] == "%"):
        i += 1
    nr, nc, nnz = (int(x) for x in lines[i].split()[:3])
    if nr != nc:
        raise RuntimeError(f"{path}:{i + 1}: adjacency matrix must be square")
    src, dst, w = [], [], []
    seen = 0
    for j in range(i + 1, len(lines)):
        if seen >= nnz:
            break
        ln = lines[j]
        if not ln or ln[0] == "%":
            continue
        tok = ln.split()
        a, b = int(tok[0]), int(tok[1])
        v = 1.0 if pattern else float(tok[2])
        if a < 1 or a > nr or b < 1 or b > nc:
            raise RuntimeError(f"{path}:{j + 1}: index out of declared range")
        seen += 1
        src.append(a - 1)
        dst.append(b - 1)
        w.append(v)
        if symmetric and a != b:
            src.append(b - 1)
            dst.append(a - 1)
            w.append(v)
    if seen != nnz:
        raise RuntimeError(f"{path}: fewer entries than declared")
    s, d, ww = _dedup(src, dst, w)
    return {"n": nr, "src": s, "dst": d, "weight": ww}


def load_graph(path, format="edge-list"):
    return load_matrix_market(path) if format == "matrix-market" else load_edge_list(path)
