"""Run tools/probe.py against another build of libgxb200.so (A/B timing of kernel variants
in one GPU call; development aid): python tools/variant_probe.py LIB.so [probe.py args]."""

from __future__ import annotations

import os
import runpy
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2203_13005_b200 import _lib, build  # noqa: E402

_lib.LIB_PATH = os.path.abspath(sys.argv[1])
build.needs_build = lambda: False
sys.argv = [os.path.join(os.path.dirname(__file__), "probe.py")] + sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
