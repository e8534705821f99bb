"""A/B equality check of two option settings on the same graph (development aid)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2203_13005_b200 import _lib as L
from paper_2203_13005_b200.device import DeviceContext, DeviceGraph, DeviceState, run_state
from paper_2203_13005_b200.rmat import RmatParams
opt, a, b = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
scale = int(sys.argv[4]) if len(sys.argv) > 4 else 20
ctx = DeviceContext(0)
src, dst, w = ctx.rmat(RmatParams(scale=scale, seed=3))
g = DeviceGraph(ctx, src, dst, None, csr=False)
out = []
for v in (a, b):
    L.set_option(opt, v)
    s = DeviceState(g, "pagerank")
    run_state(s, 6)
    out.append(s.read_attrs())
print(json.dumps({"opt": opt, "a": a, "b": b, "identical": bool(np.array_equal(out[0], out[1])),
                  "max_abs": float(np.abs(out[0] - out[1]).max())}))
