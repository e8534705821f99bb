"""R-MAT workload parameters (include/gxb_rmat.h) and a vectorised host stream.

The reference has no R-MAT generator; this fixes one
formulation so the device generator, the host stream and the CPU oracle all see
bit-identical edges. Graph500 defaults (a, b, c) = (0.57, 0.19, 0.19); the skewed
configuration uses (0.65, 0.15, 0.15) (BASELINE.json configs[4]).
"""

from __future__ import annotations

from dataclasses import asdict, dataclass

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


@dataclass(frozen=True)
class RmatParams:
    scale: int
    edge_factor: int = 16
    seed: int = 1
    a: float = 0.57
    b: float = 0.19
    c: float = 0.19
    wmax: int = 0
    scramble: bool = True
    symmetric: bool = False

    def __post_init__(self):
        if not 1 <= self.scale <= 32:
            raise ValueError("scale must be in [1, 32]")
        if min(self.a, self.b, self.c) < 0 or self.a + self.b + self.c >= 1.0:
            raise ValueError("need a, b, c >= 0 and a + b + c < 1")

    @property
    def thresholds(self) -> tuple[int, int, int]:
        return tuple(int(p * 2 ** 32) for p in (self.a, self.b, self.c))

    @property
    def num_edges(self) -> int:
        m = self.edge_factor << self.scale
        return 2 * m if self.symmetric else m

    def c_args(self):
        ta, tb, tc = self.thresholds
        return (self.scale, self.edge_factor, self.seed, ta, tb, tc, self.wmax, int(self.scramble),
                int(self.symmetric))

    def as_dict(self):
        return asdict(self)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    x = x + np.uint64(0x9E3779B97F4A7C15)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def _mix(seed: int, salt: int) -> np.uint64:
    with np.errstate(over="ignore"):
        return _splitmix64(np.array([np.uint64(seed) ^ np.uint64(salt)], dtype=np.uint64))[0]


def _scramble(x: np.ndarray, scale: int, seedmix: np.uint64) -> np.ndarray:
    mask = np.uint64((1 << scale) - 1) if scale < 64 else _M64
    sh = np.uint64((scale + 1) // 2)
    x = (x ^ (seedmix >> np.uint64(7))) & mask
    x = (x * np.uint64(0x9E3779B97F4A7C15)) & mask
    x ^= x >> sh
    x = (x * np.uint64(0xC2B2AE3D27D4EB4F)) & mask
    x ^= x >> sh
    return x & mask


def rmat_host(p: RmatParams, chunk: int = 1 << 22):
    """Host edge stream identical to the device generator; returns (src, dst, w|None) as uint32."""
    m = p.edge_factor << p.scale
    ta, tb, tc = (np.uint32(t) for t in p.thresholds)
    tab, tabc = np.uint64(int(ta) + int(tb)), np.uint64(int(ta) + int(tb) + int(tc))
    seedmix = _mix(p.seed, 0xD1B54A32D192ED03)
    wseedmix = _mix(p.seed, 0x8CB92BA72F3D8DD7)
    n = 2 * m if p.symmetric else m
    src = np.empty(n, dtype=np.uint32)
    dst = np.empty(n, dtype=np.uint32)
    w = np.empty(n, dtype=np.uint32) if p.wmax else None
    with np.errstate(over="ignore"):
        for lo in range(0, m, chunk):
            hi = min(m, lo + chunk)
            i = np.arange(lo, hi, dtype=np.uint64)
            s = np.zeros(hi - lo, dtype=np.uint64)
            d = np.zeros(hi - lo, dtype=np.uint64)
            r = None
            for level in range(p.scale):
                if level % 2 == 0:
                    r = _splitmix64(seedmix + ((i << np.uint64(4)) | np.uint64(level >> 1)))
                    u = r & np.uint64(0xFFFFFFFF)
                else:
                    u = r >> np.uint64(32)
                row = u >= tab                     # quadrants (1,0) and (1,1)
                col = ((u >= np.uint64(int(ta))) & (u < tab)) | (u >= tabc)
                s |= row.astype(np.uint64) << np.uint64(level)
                d |= col.astype(np.uint64) << np.uint64(level)
            if p.scramble:
                s = _scramble(s, p.scale, seedmix)
                d = _scramble(d, p.scale, seedmix)
            src[lo:hi] = s
            dst[lo:hi] = d
            if w is not None:
                w[lo:hi] = (np.uint64(1) + _splitmix64(wseedmix + i) % np.uint64(p.wmax)).astype(np.uint32)
    if p.symmetric:
        src[m:] = dst[:m]
        dst[m:] = src[:m]
        if w is not None:
            w[m:] = w[:m]
    return src, dst, w


GRAPH500 = dict(a=0.57, b=0.19, c=0.19)
SKEWED = dict(a=0.65, b=0.15, c=0.15)
