"""Graph input surface of the reference (`A/graph.py`), host side.

The reference keeps per-node Python tables (`Partition`, `PartitionedGraph`,
A/graph.py:93-128); here the tables live on the device (libgxb200's CSC/CSR
store), so the host only needs the edge-list container and the loader. The
loader keeps the reference's exact parsing rules and error messages
(`load_edge_list`, A/graph.py:131-166).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class GraphParseError(ValueError):
    """Raised for malformed edge-list input; carries the 1-based line number (A/graph.py:17-22)."""

    def __init__(self, lineno: int, message: str):
        super().__init__(f"line {lineno}: {message}")
        self.lineno = lineno


@dataclass(frozen=True, slots=True)
class Edge:
    src: int
    dst: int
    weight: float = 1.0


def load_edge_list(path) -> tuple[set[int], list[Edge]]:
    """Parse `src dst [weight]` lines; '#' comments, blank lines, LF/CRLF; duplicates kept."""
    vertices: set[int] = set()
    edges: list[Edge] = []
    with open(path, "r", encoding="ascii") as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split()
            if len(parts) not in (2, 3):
                raise GraphParseError(lineno, f"expected 2 or 3 fields, got {len(parts)}")
            try:
                src = int(parts[0])
                dst = int(parts[1])
            except ValueError:
                raise GraphParseError(lineno, f"non-integer vertex id in {parts[:2]}") from None
            if src < 0 or dst < 0:
                raise GraphParseError(lineno, "vertex ids must be non-negative")
            weight = 1.0
            if len(parts) == 3:
                try:
                    weight = float(parts[2])
                except ValueError:
                    raise GraphParseError(lineno, f"non-numeric weight {parts[2]!r}") from None
                if weight < 0:
                    raise GraphParseError(lineno, f"negative weight {weight}")
            vertices.add(src)
            vertices.add(dst)
            edges.append(Edge(src, dst, weight))
    return vertices, edges


def even_sizes(n: int, m: int) -> list[int]:
    """Split n items into m near-equal contiguous chunk sizes (A/graph.py:169-172)."""
    base, rem = divmod(n, m)
    return [base + (1 if j < rem else 0) for j in range(m)]


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
        """From reference-style Edge objects (or (src, dst[, w]) tuples)."""
        n = len(edges)
        src = np.empty(n, dtype=np.uint64)
        dst = np.empty(n, dtype=np.uint64)
        w = np.empty(n, dtype=np.float64)
        weighted = False
        for i, e in enumerate(edges):
            if isinstance(e, Edge):
                s, d, x = e.src, e.dst, e.weight
            else:
                s, d = e[0], e[1]
                x = e[2] if len(e) > 2 else 1.0
            src[i], dst[i], w[i] = s, d, x
            weighted |= x != 1.0
        if n and (src.max() >= 0xFFFFFFFF or dst.max() >= 0xFFFFFFFF):
            raise ValueError("vertex ids must be < 2^32 - 1 on the device")
        return cls(src.astype(np.uint32), dst.astype(np.uint32), w if weighted else None)

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
    _, edges = load_edge_list(text_path)
    ea = EdgeArrays.from_edges(edges)
    write_edge_binary(bin_path, ea)
    return len(ea)
