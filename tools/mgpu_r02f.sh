#!/bin/bash
set -u
O=gpurun_out/mg7
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
p=30110
timeout 600 python -m pytest tests/test_mp_ipc_gpu.py tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_api_gpu.py tests/test_gpu_edges.py -q -x -k "not golden_vectors" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
python tools/probe.py --scale 24 --algo lp --a 0.65 --iters 15 > $O/lp24.json
for n in 2 4; do
  p=$((p+1)); timeout 300 $TR --nproc-per-node $n --master-port $p tools/mgpu_rounds.py sssp 26 2>&1 | grep "{" > $O/rounds_sssp_n$n.log; echo "rounds n=$n rc=$?"
  for w in sssp-s26 cc-s24 lp-s22; do
    st=12; [ $w = cc-s24 ] && st=8; [ $w = lp-s22 ] && st=15
    p=$((p+1)); timeout 600 $TR --nproc-per-node $n --master-port $p bench.py --gpus $n --workload $w --steps $st --warmup 3 --no-e2e --no-parity > $O/wl_${w}_n${n}.json 2> $O/wl_${w}_n${n}.err; echo "wl $w n=$n rc=$?"
  done
  p=$((p+1)); timeout 600 $TR --nproc-per-node $n --master-port $p tools/mgpu_check.py --scale 22 > $O/check_s22_n$n.log 2>&1; echo "check n=$n rc=$?"
done
python bench.py --workload lp-s22 --steps 15 --warmup 3 --no-e2e --no-parity --no-cpu-baseline --no-python-reference > $O/wl_lp-s22_n1.json 2> $O/wl_lp-s22_n1.err
python bench.py --workload cc-s24 --steps 8 --warmup 3 --no-e2e --no-parity --no-cpu-baseline --no-python-reference > $O/wl_cc-s24_n1.json 2> $O/wl_cc-s24_n1.err
python bench.py --workload sssp-s26 --steps 12 --warmup 3 --no-e2e --no-parity --no-cpu-baseline --no-python-reference > $O/wl_sssp-s26_n1.json 2> $O/wl_sssp-s26_n1.err
