#!/bin/bash
set -u
O=gpurun_out/mg8
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
p=30210
timeout 300 python -m pytest tests/test_mp_ipc_gpu.py -q -x > $O/mp.log 2>&1; echo "mp rc=$?"
for n in 2 4; do
  p=$((p+1)); timeout 300 $TR --nproc-per-node $n --master-port $p tools/mgpu_rounds.py sssp 26 2>&1 | grep "{" > $O/rounds_sssp_n$n.log; echo "rounds n=$n rc=$?"
  for w in sssp-s26 cc-s24; do
    st=12; [ $w = cc-s24 ] && st=8
    p=$((p+1)); timeout 600 $TR --nproc-per-node $n --master-port $p bench.py --gpus $n --workload $w --steps $st --warmup 3 --no-e2e --no-parity > $O/wl_${w}_n${n}.json 2> $O/wl_${w}_n${n}.err; echo "wl $w n=$n rc=$?"
  done
  p=$((p+1)); timeout 600 $TR --nproc-per-node $n --master-port $p tools/mgpu_check.py --scale 22 > $O/check_s22_n$n.log 2>&1; echo "check n=$n rc=$?"
  p=$((p+1)); timeout 1200 $TR --nproc-per-node $n --master-port $p bench.py --gpus $n --steps 20 --warmup 3 > $O/bench_n$n.json 2> $O/bench_n$n.err; echo "bench n=$n rc=$?"
done
