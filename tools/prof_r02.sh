#!/bin/bash
# Round-2 evidence captures on one B200 (each program first runs clean without ncu).
# Usage: bash tools/prof_r02.sh [step...]; outputs in gpurun_out/r02/
set -u
O=gpurun_out/r02
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
run() { echo "== $*" >> $O/log.txt; "$@" >> $O/log.txt 2>&1; echo "rc=$?" >> $O/log.txt; }
for step in "$@"; do
case $step in
lp)
  run python tools/probe.py --scale 24 --algo lp --a 0.65 --iters 15
  run $NCU -k regex:k_lp_pull -s 3 -c 1 -o $O/lp24_pull python tools/probe.py --scale 24 --algo lp --a 0.65 --iters 6
  run $NCU -k regex:k_lp_push -s 1 -c 1 -o $O/lp24_push python tools/probe.py --scale 24 --algo lp --a 0.65 --iters 15 ;;
cc)
  run python tools/probe.py --scale 24 --algo cc --iters 20
  run $NCU -k regex:k_tile_a -s 1 -c 1 -o $O/cc24_tile python tools/probe.py --scale 24 --algo cc --iters 4 ;;
sssp)
  run python tools/probe.py --scale 24 --algo sssp --iters 30
  run $NCU -k regex:"k_push<" -s 1 -c 1 -o $O/sssp24_push python tools/probe.py --scale 24 --algo sssp --iters 30
  run $NCU -k regex:k_push_rowpre -s 2 -c 1 -o $O/sssp24_rowpre python tools/probe.py --scale 24 --algo sssp --iters 30 ;;
pack)
  run python tools/probe_parts.py --scale 20 --algo cc --parts 2
  run $NCU -k regex:"k_pack|k_unpack" -s 2 -c 2 -o $O/cc20_pack python tools/probe_parts.py --scale 20 --algo cc --parts 2 ;;
sanitizer)
  run timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "s10_seed11 or s12_seed12" -p no:cacheprovider
  run timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "s10_seed11 and (sssp or cc) and auto" -p no:cacheprovider ;;
esac
done
