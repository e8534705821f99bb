"""Graph input surface of the reference (`A/graph.py`), host side.

The reference keeps per-node Python tables (`Partition`, `PartitionedGraph`,
A/graph.py:93-128); here the tables live on the device (libgxb200's CSC/CSR
store), so the host only needs columnar edge arrays: a text reader with the
reference's parsing rules and error messages (`load_edge_list`, A/graph.py:131-166)
and a memory-mapped binary format for ingest at scale.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class GraphParseError(ValueError):
    """Malformed edge-list input; `lineno` is 1-based (the reference's GraphParseError,
    A/graph.py:17-22, same message format)."""

    def __init__(self, lineno: int, message: str):
        super().__init__(f"line {lineno}: {message}")
        self.lineno = lineno


def _first_error(lineno: int, fields: list[str]) -> str | None:
    """The reference's per-line checks, in its order (A/graph.py:146-162)."""
    if len(fields) not in (2, 3):
        return f"expected 2 or 3 fields, got {len(fields)}"
    try:
        a, b = int(fields[0]), int(fields[1])
    except ValueError:
        return f"non-integer vertex id in {fields[:2]}"
    if a < 0 or b < 0:
        return "vertex ids must be non-negative"
    if len(fields) == 3:
        try:
            x = float(fields[2])
        except ValueError:
            return f"non-numeric weight {fields[2]!r}"
        if x < 0:
            return f"negative weight {x}"
    return None


def read_edge_text(path) -> "EdgeArrays":
    """Columnar reader of the reference's text edge list (`src dst [weight]` per line,
    '#' comments, blank lines, LF / CRLF, duplicates and self-loops kept in file order):
    the same accepted inputs, values and errors as `load_edge_list` (A/graph.py:131-166,
    pinned by tests/golden/edge_lists.json), straight into the device ingest columns.

    Lines are tokenised once; ids and weights are converted column-wise, and only when a
    conversion or range check fails is the offending line located (the first one in file
    order) and diagnosed with the reference's message."""
    with open(path, "r", encoding="ascii") as fh:
        text = fh.read()
    rows = [(n, ln.split()) for n, ln in enumerate(text.split("\n"), start=1)]
    rows = [(n, f) for n, f in rows if f and not f[0].startswith("#")]
    widths = {len(f) for _, f in rows}
    try:
        if not widths <= {2, 3}:
            raise ValueError
        src = np.array([int(f[0]) for _, f in rows], dtype=np.int64)
        dst = np.array([int(f[1]) for _, f in rows], dtype=np.int64)
        w = np.array([float(f[2]) if len(f) == 3 else 1.0 for _, f in rows], dtype=np.float64)
        if (src < 0).any() or (dst < 0).any() or (w < 0).any():
            raise ValueError
    except (ValueError, OverflowError):
        for n, f in rows:
            msg = _first_error(n, f)
            if msg is not None:
                raise GraphParseError(n, msg) from None
        raise
    weighted = bool((w != 1.0).any())
    if src.size and max(src.max(), dst.max()) >= 0xFFFFFFFF:
        raise ValueError("vertex ids must be < 2^32 - 1 on the device")
    return EdgeArrays(src.astype(np.uint32), dst.astype(np.uint32), w if weighted else None)


@dataclass
class EdgeArrays:
    """Columnar edge list (the device ingest format): uint32 ids, float64 weights or None."""

    src: np.ndarray
    dst: np.ndarray
    weight: np.ndarray | None = None

    def __post_init__(self):
        self.src = np.ascontiguousarray(self.src, dtype=np.uint32)
        self.dst = np.ascontiguousarray(self.dst, dtype=np.uint32)
        if self.src.shape != self.dst.shape:
            raise ValueError("src/dst length mismatch")
        if self.weight is not None:
            self.weight = np.ascontiguousarray(self.weight, dtype=np.float64)
            if self.weight.shape != self.src.shape:
                raise ValueError("weight length mismatch")

    def __len__(self) -> int:
        return int(self.src.size)

    @classmethod
    def from_edges(cls, edges) -> "EdgeArrays":
        """From reference Edge objects (`.src / .dst / .weight`, A/graph.py:39-43) or
        (src, dst[, w]) tuples."""
        def triple(e):
            if hasattr(e, "src"):
                return e.src, e.dst, e.weight
            return e[0], e[1], (e[2] if len(e) > 2 else 1.0)
        cols = np.array([triple(e) for e in edges], dtype=np.float64).reshape(-1, 3)
        src, dst, w = cols[:, 0], cols[:, 1], cols[:, 2]
        if src.size and (src.min() < 0 or dst.min() < 0 or max(src.max(), dst.max()) >= 0xFFFFFFFF):
            raise ValueError("vertex ids must be in [0, 2^32 - 1) on the device")
        return cls(src.astype(np.uint32), dst.astype(np.uint32), w.copy() if (w != 1.0).any() else None)

    def vertex_ids(self) -> np.ndarray:
        """Ids present in any edge, ascending (A/graph.py:163-164)."""
        return np.union1d(self.src, self.dst)

    def out_degree(self) -> dict[int, int]:
        """Global out-degree table over present ids (duplicates and self-loops count, A/graph.py:203-210)."""
        ids = self.vertex_ids()
        cnt = np.zeros(ids.size, dtype=np.int64)
        np.add.at(cnt, np.searchsorted(ids, self.src), 1)
        return {int(v): int(c) for v, c in zip(ids, cnt)}


# ---- binary edge format (ingest at scale without the text path) ----
#
# Layout (little endian): 32-byte header  b"GXEDGE01" | u64 num_edges | u32 flags | u32 0,
# then src u32[E], dst u32[E] and, when flags & 1, weights f64[E]. The arrays are read as
# memory maps, so a 1 G-edge file feeds DeviceGraph (which copies host arrays once to HBM)
# without a per-edge Python object (the text loader costs ~190 B and ~5 µs per edge).
EDGE_MAGIC = b"GXEDGE01"
_HEADER = np.dtype([("magic", "S8"), ("num_edges", "<u8"), ("flags", "<u4"), ("pad", "<u4"),
                    ("reserved", "<u8")])


def write_edge_binary(path, edges: "EdgeArrays") -> None:
    """Write an EdgeArrays in the binary edge format."""
    h = np.zeros(1, dtype=_HEADER)
    h["magic"] = EDGE_MAGIC
    h["num_edges"] = len(edges)
    h["flags"] = 1 if edges.weight is not None else 0
    with open(path, "wb") as fh:
        fh.write(h.tobytes())
        fh.write(np.ascontiguousarray(edges.src, dtype="<u4").tobytes())
        fh.write(np.ascontiguousarray(edges.dst, dtype="<u4").tobytes())
        if edges.weight is not None:
            fh.write(np.ascontiguousarray(edges.weight, dtype="<f8").tobytes())


def read_edge_binary(path) -> "EdgeArrays":
    """Read the binary edge format (memory-mapped columns); raises GraphParseError (line 0)
    for a malformed file."""
    import os
    size = os.path.getsize(path)
    if size < _HEADER.itemsize:
        raise GraphParseError(0, "binary edge file shorter than its header")
    h = np.fromfile(path, dtype=_HEADER, count=1)[0]
    if bytes(h["magic"]) != EDGE_MAGIC:
        raise GraphParseError(0, "not a GXEDGE01 binary edge file")
    n, weighted = int(h["num_edges"]), bool(int(h["flags"]) & 1)
    need = _HEADER.itemsize + 8 * n + (8 * n if weighted else 0)
    if size != need:
        raise GraphParseError(0, f"binary edge file has {size} bytes, expected {need} for {n} edges")
    off = _HEADER.itemsize
    src = np.memmap(path, dtype="<u4", mode="r", offset=off, shape=(n,)) if n else np.empty(0, np.uint32)
    dst = np.memmap(path, dtype="<u4", mode="r", offset=off + 4 * n, shape=(n,)) if n else np.empty(0, np.uint32)
    w = None
    if weighted:
        w = np.memmap(path, dtype="<f8", mode="r", offset=off + 8 * n, shape=(n,)) if n else np.empty(0)
    return EdgeArrays(src, dst, w)


def edge_list_to_binary(text_path, bin_path) -> int:
    """Convert a reference text edge list (load_edge_list rules) to the binary format."""
    ea = read_edge_text(text_path)
    write_edge_binary(bin_path, ea)
    return len(ea)
