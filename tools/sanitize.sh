#!/bin/bash
# compute-sanitizer over small parity cases (S <= 12): memcheck on every kernel family,
# racecheck / synccheck on the shared-memory kernels (tile folds, LP tables, scans).
set -u
O=gpurun_out/san
mkdir -p $O
CS="compute-sanitizer --error-exitcode 9 --print-limit 20"
K='s10_seed11 or golden_vectors and (path3 or ring12 or random20w or sparse_ids)'
timeout 1500 $CS --tool memcheck python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$K" > $O/memcheck_parity.log 2>&1; echo "memcheck parity rc=$?"
timeout 900 $CS --tool memcheck python -m pytest tests/test_gpu_edges.py -q -x -p no:cacheprovider -k "not 300k and not hub" > $O/memcheck_edges.log 2>&1; echo "memcheck edges rc=$?"
timeout 900 $CS --tool memcheck python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "peer_delta and 2-edges or owned_install and 2-" > $O/memcheck_exchange.log 2>&1; echo "memcheck exchange rc=$?"
timeout 1500 $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "s10_seed11 and auto" > $O/racecheck.log 2>&1; echo "racecheck rc=$?"
timeout 900 $CS --tool synccheck python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "s10_seed11 and auto" > $O/synccheck.log 2>&1; echo "synccheck rc=$?"
for f in $O/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|passed|failed" $f | tail -3; done
