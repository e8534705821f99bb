"""Run bench.py against another build of libgxb200.so (A/B of kernel variants under the
same launcher, torchrun included; development aid): python tools/variant_bench.py LIB.so
[bench.py args]."""

from __future__ import annotations

import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2203_13005_b200 import _lib, build  # noqa: E402

_lib.LIB_PATH = os.path.abspath(sys.argv[1])
build.needs_build = lambda: False
sys.argv = [os.path.join(ROOT, "bench.py")] + sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
