#!/bin/bash
# Round-2 multi-GPU runs (second pass, per-peer delta exchange): parity vs the oracle,
# frontier workloads (one run each), PageRank bench lines with NVLink counters around them.
set -u
O=gpurun_out/mg2
mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
p=29700
nvl() { nvidia-smi nvlink -gt d > $O/$1 2>&1 || true; }
for n in 2 4; do
  [ $n -le $NG ] || continue
  p=$((p+1)); timeout 600 $TR --nproc-per-node $n --master-port $p tools/mgpu_check.py --scale 20 > $O/check_s20_n$n.log 2>&1; echo "check n=$n rc=$?"
  for w in sssp-s26 cc-s24 lp-s22; do
    st=12; [ $w = cc-s24 ] && st=8; [ $w = lp-s22 ] && st=15
    p=$((p+1)); timeout 600 $TR --nproc-per-node $n --master-port $p bench.py --gpus $n --workload $w --steps $st --warmup 3 --no-e2e --no-parity > $O/wl_${w}_n$n.json 2> $O/wl_${w}_n$n.err; echo "wl $w n=$n rc=$?"
  done
  nvl nvl_before_n$n.txt
  p=$((p+1)); timeout 1200 $TR --nproc-per-node $n --master-port $p bench.py --gpus $n --steps 20 --warmup 3 > $O/bench_n$n.json 2> $O/bench_n$n.err; echo "bench n=$n rc=$?"
  nvl nvl_after_n$n.txt
done
