"""Convert a reference text edge list to the binary GXEDGE01 format (graph.write_edge_binary).

    python tools/edges2bin.py graph.txt graph.gxe
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2203_13005_b200.graph import edge_list_to_binary  # noqa: E402

if __name__ == "__main__":
    if len(sys.argv) != 3:
        sys.exit(__doc__)
    print(f"{edge_list_to_binary(sys.argv[1], sys.argv[2])} edges written to {sys.argv[2]}")
