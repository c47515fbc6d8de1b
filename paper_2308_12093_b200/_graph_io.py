"""Graph file ingestion (graph.hpp:57-147): whitespace edge lists
("src dst [weight]", '#' comments, node count = max index + 1) and
MatrixMarket coordinate files; edges deduplicated keeping the last weight and
returned in canonical (src, dst) order.  Host-side I/O, not on the device path.
"""
from __future__ import annotations

import re

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


class _Line:
    """Token extraction with the reference's std::istringstream semantics
    (graph.hpp:68-78): `>>` skips whitespace, then reads the longest numeric
    prefix; a failed read leaves the stream failed (value 0 for a started but
    malformed number, unchanged at end of line) and later reads fail too."""

    _INT = re.compile(r"\s*([+-]?\d+)")
    _DBL = re.compile(r"\s*([+-]?(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?)")
    _TOK = re.compile(r"\s*(\S+)")

    def __init__(self, text):
        self.s, self.pos, self.ok = text, 0, True

    def _take(self, rx):
        if not self.ok:
            return None
        m = rx.match(self.s, self.pos)
        if m is None:
            self.ok = False
            return None
        self.pos = m.end()
        return m.group(1)

    def int(self):
        t = self._take(self._INT)
        if t is not None and not -(1 << 63) <= int(t) < (1 << 63):
            self.ok = False
            return None
        return None if t is None else int(t)

    def double(self, default):
        """`ls >> w`: default kept at end of line, 0.0 on a malformed number."""
        if not self.ok:
            return default
        if self.s[self.pos:].strip() == "":
            self.ok = False
            return default
        t = self._take(self._DBL)
        return 0.0 if t is None else float(t)

    def token(self):
        return self._take(self._TOK)


def load_edge_list(path):
    src, dst, w = [], [], []
    max_idx = -1
    try:
        fh = open(path)
    except OSError:
        raise RuntimeError(f"cannot open {path}") from None
    with fh:
        for line_no, line in enumerate(fh, 1):
            ls = _Line(line.rstrip("\n").split("#", 1)[0])
            s = ls.int()
            if s is None:
                continue  # blank, comment-only or header line (graph.hpp:76)
            d = ls.int()
            if d is None:
                raise RuntimeError(f"{path}:{line_no}: expected 'src dst [weight]'")
            wt = ls.double(1.0)
            if ls.token() is not None:
                raise RuntimeError(f"{path}:{line_no}: trailing tokens")
            if s < 0 or d < 0:
                raise RuntimeError(f"{path}:{line_no}: negative node index")
            src.append(s)
            dst.append(d)
            w.append(wt)
            max_idx = max(max_idx, s, d)
    s, d, ww = _dedup(src, dst, w)
    return {"n": max_idx + 1, "src": s, "dst": d, "weight": ww}


def load_matrix_market(path):
    try:
        fh = open(path)
    except OSError:
        raise RuntimeError(f"cannot open {path}") from None
    with fh:
        lines = fh.read().split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    if not lines:
        raise RuntimeError(f"{path}: empty file")
    head = lines[0].split()
    head += [""] * (5 - len(head))
    if head[0] != "%%MatrixMarket" or head[1] != "matrix" or head[2] != "coordinate":
        raise RuntimeError(f"{path}:1: expected a MatrixMarket coordinate header")
    field, symmetry = head[3], head[4]
    pattern = field == "pattern"
    symmetric = symmetry in ("symmetric", "skew-symmetric")
    if field not in ("real", "integer") and not pattern:
        raise RuntimeError(f"{path}:1: unsupported field type '{field}'")
    nr = nc = nnz = 0
    i = 1
    line_no = 1
    while i < len(lines):
        line_no = i + 1
        ln = lines[i]
        i += 1
        if not ln or ln[0] == "%":
            continue
        ls = _Line(ln)
        vals = (ls.int(), ls.int(), ls.int())
        if None in vals:
            raise RuntimeError(f"{path}:{line_no}: expected 'rows cols nnz'")
        nr, nc, nnz = vals
        break
    if nr != nc:
        raise RuntimeError(f"{path}:{line_no}: adjacency matrix must be square")
    src, dst, w = [], [], []
    seen = 0
    for j in range(i, len(lines)):
        if seen >= nnz:
            break
        ln = lines[j]
        if not ln or ln[0] == "%":
            continue
        ls = _Line(ln)
        a, b = ls.int(), ls.int()
        if a is None or b is None:
            raise RuntimeError(f"{path}:{j + 1}: expected 'i j [value]'")
        v = 1.0
        if not pattern:
            v = ls.double(None)
            if not ls.ok:
                raise RuntimeError(f"{path}:{j + 1}: missing value")
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
