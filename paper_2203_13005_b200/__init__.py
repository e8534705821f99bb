"""gx-b200: B200-native GX-Plug per-iteration graph compute path (arXiv 2203.13005).

Drop-in for the reference's algorithm-template / daemon / agent interfaces
(`pkg/src/accelgraph`), executing MSGGen -> MSGMerge -> MSGApply and the mirror
exchange in hand-written sm_100a kernels (libgxb200.so, include/gxb.h).
"""

__version__ = "0.1.0"
